"""One training step of a config between cudaProfilerStart/Stop, for ncu --profile-from-start off
(the --set full captures behind bench.py's roofline.traffic):

  BLSTM_OVERLAP=0 ncu --profile-from-start off --set full -k regex:"gemm_f16|lstm_rec" \
      -o gpurun_out/r02_full_C3 python scripts/ncu_step.py --config C3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1608_00895_b200 import synth  # noqa: E402
from paper_1608_00895_b200.train import StackTrainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    cfg, params, batch = synth.make_workload(synth.CONFIGS[a.config])
    tr = StackTrainer(cfg, params, batch, dev)
    for _ in range(a.warmup):
        tr.step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    tr.step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("valid frames", tr.valid_frames)


if __name__ == "__main__":
    main()
