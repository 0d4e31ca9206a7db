"""Bandwidth of blstm_gather_chunks (NEXT-4): one C3-shaped batch (T=250, B=81, D=40) gathered
from a device-resident corpus of overlapping chunks (C=250, S=125).  Algorithmic bytes per
batch: x read + written (2 x T*B*D*4 over valid frames, the padding written only), mask and
labels (T*B*(1+4+4))."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1608_00895_b200 import blstm, data  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    dev = torch.device("cuda:0")
    g = np.random.default_rng(0)
    lengths = np.clip(np.rint(g.normal(738, 291, size=2000)), 50, 2500).astype(int)
    xs = [g.standard_normal((L, 40)).astype(np.float32) for L in lengths]
    ls = [g.integers(0, 1501, size=L).astype(np.int32) for L in lengths]
    corpus = data.DeviceCorpus(xs, ls, dev)
    batches = data.make_batches(data.chunk_sequences(lengths, 250, 125), 81, seed=1)
    T, B, D = 250, 81, 40
    x = torch.empty((T, B, D), device=dev)
    m = torch.empty((T, B), dtype=torch.uint8, device=dev)
    lab = torch.empty((T, B), dtype=torch.int32, device=dev)
    nb = corpus.plan_epoch(batches, B, T)
    for k in range(5):
        corpus.gather_planned(k, x, m, lab)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 200
    e0.record()
    for k in range(K):
        corpus.gather_planned(k % nb, x, m, lab)
    e1.record()
    torch.cuda.synchronize()
    us_call = e0.elapsed_time(e1) * 1e3 / K
    blstm.blstm_profile_enable(2)  # device time of the gather kernels alone
    for k in range(K):
        corpus.gather_planned(k % nb, x, m, lab)
    torch.cuda.synchronize()
    recs = blstm.blstm_profile_timeline()
    blstm.blstm_profile_enable(0)
    us = 1e3 * sum(r[3] - r[2] for r in recs) / len(recs)
    valid = np.mean([data.chunk_frames([b]) for b in batches[:K]])
    byts = valid * D * 4 + T * B * D * 4 + T * B * (1 + 4) + valid * 4
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    print(json.dumps(dict(corpus_frames=corpus.corpus_frames(), chunk_frames_epoch=data.chunk_frames(batches),
                          batches=len(batches), us_per_batch=round(us, 2), us_per_call_from_python=round(us_call, 2), bytes_per_batch=int(byts),
                          gbs=round(byts / us / 1e3, 1), frac_hbm=round(byts / us / 1e3 / peak, 3),
                          note="kernel device time (CUDA events around each launch); epoch chunk table resident on the device (plan_epoch); the per-call figure includes the Python binding's launch overhead")))


if __name__ == "__main__":
    main()
