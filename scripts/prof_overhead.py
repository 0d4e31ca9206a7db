"""Step time with and without the per-launch CUDA-event scopes (blstm_profile_enable) that bench.py
keeps on over its timed region: the cost of the roofline instrumentation itself."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1608_00895_b200 import blstm, synth  # noqa: E402
from paper_1608_00895_b200.train import DPSchedule, StackTrainer, dp_comm_from_torch  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    dev = torch.device("cuda:0")
    cfg, params, batch = synth.make_workload(synth.CONFIGS[name], 0)
    tr = StackTrainer(cfg, params, batch, dev, lr=1e-5, comm=dp_comm_from_torch(0, 1), world=1, sched=DPSchedule("sync", 1))
    smi = None
    if "--smi" in sys.argv:  # bench.py's clock sampler running beside the steps
        import subprocess
        smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=timestamp,clocks.sm,power.draw",
                                "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.DEVNULL)
    for _ in range(5):
        tr.step()
    torch.cuda.synchronize()
    for rnd in range(3):
        for on in (1, 0):
            blstm.blstm_profile_enable(bool(on))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(steps):
                tr.step()
            e1.record()
            torch.cuda.synchronize()
            blstm.blstm_profile_enable(False)
            print(f"{name} profile={'on ' if on else 'off'} smi={smi is not None} {e0.elapsed_time(e1) / steps:.4f} ms/step",
                  flush=True)
    if smi is not None:
        smi.terminate()


if __name__ == "__main__":
    main()
