"""The default stack step under serialized execution.

The forward recurrence spins on Z tiles of a GEMM launched beside it as a programmatic
dependent.  When something keeps that GEMM off the GPU until the recurrence
exits (a profiler replaying kernels one at a time, CUDA_LAUNCH_BLOCKING=1, an MPS SM cap, a
co-tenant), the start arbitration (common.cuh arb_decide) makes the recurrence exit and a
conditional re-launch after the GEMM run the layer.  Here each variant runs in its own process
(the library reads its environment once): the default, CUDA_LAUNCH_BLOCKING=1 (auto-detected:
no overlap), CUDA_LAUNCH_BLOCKING=1 with the overlap forced on (BLSTM_OVERLAP=2: the abort path
runs for every layer) and BLSTM_OVERLAP=0.  All four must give bit-identical loss and gradients,
and the forced one must not hang."""
import hashlib
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1608_00895_b200 import blstm, synth
L, D, H, K, T, B = 3, 40, 200, 17, 40, 37
lengths = np.array([40 - (i * 7) % 33 for i in range(B)], np.int32)
params = synth.stack_params(L, D, H, K)
batch = synth.speech_batch(T, B, D, K, lengths, seed=1000)
desc = blstm.stack_desc(L, D, H, K, T, B)
n, offs = blstm.blstm_param_offsets(desc)
dev = torch.device("cuda:0")
theta = torch.zeros(n, dtype=torch.float32, device=dev)
for l, (f, bw) in enumerate(params.layers):
    for d, p in enumerate((f, bw)):
        e = 6 * l + 3 * d
        for q, a in enumerate((p.W, p.R, p.b)):
            theta[offs[e + q]: offs[e + q] + a.size] = torch.tensor(a.ravel(), dtype=torch.float32)
theta[offs[6 * L]: offs[6 * L] + params.W_out.size] = torch.tensor(params.W_out.ravel(), dtype=torch.float32)
theta[offs[6 * L + 1]: offs[6 * L + 1] + K] = torch.tensor(params.b_out, dtype=torch.float32)
grad = torch.zeros(n, dtype=torch.float32, device=dev)
ws = torch.empty(blstm.blstm_stack_workspace_bytes(desc), dtype=torch.uint8, device=dev)
loss = torch.zeros(1, dtype=torch.float64, device=dev)
ferr = torch.zeros(1, dtype=torch.int32, device=dev)
side = torch.cuda.Stream()
for _ in range(2):
    grad.zero_()
    blstm.blstm_stack_fwd_bwd(desc, theta, grad, torch.tensor(batch.x, device=dev), torch.tensor(batch.mask, device=dev),
                              torch.tensor(batch.labels, device=dev), None, loss, ferr, None, ws, s_side=side)
torch.cuda.synchronize()
h = hashlib.sha256(grad.cpu().numpy().tobytes() + loss.cpu().numpy().tobytes()).hexdigest()
print("RESULT", h, float(loss.item()), int(ferr.item()))
"""


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT")][-1]
    return line.split()[1:]


def test_serialized_execution_is_correct_and_bitwise_equal():
    base = _run({})
    assert _run({"CUDA_LAUNCH_BLOCKING": "1"}) == base
    assert _run({"CUDA_LAUNCH_BLOCKING": "1", "BLSTM_OVERLAP": "2"}) == base  # abort + re-launch path
    assert _run({"BLSTM_OVERLAP": "0"}) == base
