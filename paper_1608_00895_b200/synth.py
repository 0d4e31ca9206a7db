"""Seeded synthetic workloads shared by the CUDA path, the oracle and the bench.

This module holds NO arithmetic of the method (no LSTM, no loss, no update):
it only draws inputs and initial parameters, as fp32 numpy arrays, so that the
oracle (fp64, oracle/) and the CUDA path (paper_1608_00895_b200/) consume the
same bytes.  Recipe: SURVEY.md §8(d) "Concrete synthetic inputs", restated in
DESIGN.md §3.

Workload shapes follow the paper's CHiME setup (§6):
"chunks of 250 frames", "81 chunks" per batch, "1501" output classes; the
feature width is BASELINE.json's 40 (reading R12).  Sequence lengths
are ``round(N(738, 291))`` clipped to [50, 2500] (reading R13).
Chunking (§4) is used only to shape the batch.

Layouts (time-major, row-major, §5):
  x      [T, B, D]  float32, zero at padded frames
  mask   [T, B]     uint8 in {0, 1}, trailing padding
  labels [T, B]     int32 in [0, K), 0 at padded frames
Parameters per layer and direction (SPEC S:171 gate blocks i|f|g|o):
  W [D_l, 4H], R [H, 4H], b [4H];  head W_out [2H, K], b_out [K].
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

PARAM_SEED = 1
DATA_SEED_BASE = 1000

CHUNK = 250            # PAPER.md P:293 "chunks of 250 frames"
CHUNKS_PER_BATCH = 81
N_CLASSES = 1501


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


@dataclass
class LayerParams:
    W: np.ndarray  # [D_l, 4H]
    R: np.ndarray  # [H, 4H]
    b: np.ndarray  # [4H]


@dataclass
class StackParams:
    layers: List[Tuple[LayerParams, LayerParams]]  # (fwd, bwd) per layer
    W_out: Optional[np.ndarray] = None             # [2H, K]
    b_out: Optional[np.ndarray] = None             # [K]


@dataclass
class Batch:
    x: np.ndarray            # [T, B, D] float32
    mask: np.ndarray         # [T, B] uint8
    labels: Optional[np.ndarray] = None  # [T, B] int32
    dy_top: Optional[np.ndarray] = None  # [T, B, 2H] float32 (no-head workloads)
    lengths: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))


def _uniform(g: np.random.Generator, shape, fan_in: int, fan_out: int) -> np.ndarray:
    # SPEC S:147 init rule (reading R11)
    a = np.sqrt(6.0 / (fan_in + fan_out))
    return g.uniform(-a, a, size=shape).astype(np.float32)


def lstm_params(g: np.random.Generator, D: int, H: int) -> LayerParams:
    W = _uniform(g, (D, 4 * H), D, 4 * H)
    R = _uniform(g, (H, 4 * H), H, 4 * H)
    b = np.zeros(4 * H, np.float32)
    b[H:2 * H] = 1.0  # forget-gate bias +1
    return LayerParams(W, R, b)


def stack_params(L: int, D: int, H: int, K: int, bidirectional: bool = True,
                 seed: int = PARAM_SEED) -> StackParams:
    g = rng(seed)
    layers = []
    for l in range(L):
        Dl = D if l == 0 else (2 * H if bidirectional else H)
        fwd = lstm_params(g, Dl, H)
        bwd = lstm_params(g, Dl, H) if bidirectional else None
        layers.append((fwd, bwd))
    W_out = b_out = None
    if K > 0:
        W_out = _uniform(g, (2 * H, K), 2 * H, K)
        b_out = np.zeros(K, np.float32)
    return StackParams(layers, W_out, b_out)


def ar1_features(g: np.random.Generator, T: int, B: int, D: int,
                 lengths: np.ndarray) -> np.ndarray:
    """AR(1) per dimension, x_t = 0.9 x_{t-1} + sqrt(0.19) e_t: unit variance."""
    x = np.empty((T, B, D), np.float64)
    x[0] = g.standard_normal((B, D))
    for t in range(1, T):
        x[t] = 0.9 * x[t - 1] + np.sqrt(0.19) * g.standard_normal((B, D))
    for b, n in enumerate(lengths):
        x[n:, b, :] = 0.0  # zero at padded frames
    return x.astype(np.float32)


def mask_from_lengths(T: int, lengths: np.ndarray) -> np.ndarray:
    t = np.arange(T)[:, None]
    return (t < np.asarray(lengths)[None, :]).astype(np.uint8)


def chunked_lengths(g: np.random.Generator, n_chunks: int = CHUNKS_PER_BATCH,
                    chunk: int = CHUNK, mu: float = 738.0, sigma: float = 291.0,
                    lo: int = 50, hi: int = 2500) -> np.ndarray:
    """Valid length of each chunk in one batch.

    Sequences of length round(N(mu, sigma)) clipped to [lo, hi] are cut into
    non-overlapping chunks of `chunk` frames (chunk step = chunk size); the batch
    takes `n_chunks` chunks from a seeded shuffle of the chunk pool.
    """
    pool: List[int] = []
    while len(pool) < 4 * n_chunks:
        L = int(np.clip(np.rint(g.normal(mu, sigma)), lo, hi))
        full, rest = divmod(L, chunk)
        pool.extend([chunk] * full)
        if rest:
            pool.append(rest)
    pool_arr = np.array(pool, np.int32)
    g.shuffle(pool_arr)
    return pool_arr[:n_chunks].copy()


def speech_batch(T: int, B: int, D: int, K: int, lengths: np.ndarray,
                 seed: int) -> Batch:
    g = rng(seed)
    x = ar1_features(g, T, B, D, lengths)
    mask = mask_from_lengths(T, lengths)
    labels = g.integers(0, K, size=(T, B), dtype=np.int32) if K > 0 else None
    if labels is not None:
        labels[mask == 0] = 0
    return Batch(x=x, mask=mask, labels=labels, lengths=np.asarray(lengths, np.int32))


# ----------------------------------------------------------------------------
# The five BASELINE.json configs.
# ----------------------------------------------------------------------------

@dataclass
class Config:
    name: str
    L: int
    D: int
    H: int
    K: int          # 0 = no head (dy_top drives the backward pass)
    T: int
    B: int
    bidirectional: bool = True


CONFIGS = {
    "C1": Config("C1", L=1, D=4, H=8, K=0, T=10, B=2, bidirectional=False),
    "C2": Config("C2", L=1, D=40, H=500, K=0, T=500, B=32),
    "C3": Config("C3", L=5, D=40, H=500, K=N_CLASSES, T=CHUNK, B=CHUNKS_PER_BATCH),
    "C5": Config("C5", L=4, D=40, H=1024, K=N_CLASSES, T=1000, B=128),
}


def config_lengths(cfg: Config, seed: int) -> np.ndarray:
    g = rng(seed + 7)
    if cfg.name == "C1":
        return np.array([10, 7], np.int32)
    if cfg.name == "C2":
        lens = g.integers(100, 501, size=cfg.B).astype(np.int32)
        lens[g.integers(0, cfg.B)] = 500
        return lens
    if cfg.name == "C3":
        return chunked_lengths(g, cfg.B, cfg.T)
    if cfg.name == "C5":
        lens = np.clip(np.rint(g.normal(738.0, 291.0, size=cfg.B)), 50, cfg.T).astype(np.int32)
        lens[g.integers(0, cfg.B)] = cfg.T
        return lens
    raise KeyError(cfg.name)


def make_workload(cfg: Config, rank: int = 0, B: Optional[int] = None,
                  T: Optional[int] = None):
    """(params, batch) for a config; data seed 1000+rank, parameter seed 1."""
    import dataclasses
    if B is not None or T is not None:
        cfg = dataclasses.replace(cfg, B=B or cfg.B, T=T or cfg.T)
    seed = DATA_SEED_BASE + rank
    lengths = config_lengths(cfg, seed)
    if len(lengths) != cfg.B:
        lengths = np.resize(lengths, cfg.B)
    lengths = np.minimum(lengths, cfg.T)
    batch = speech_batch(cfg.T, cfg.B, cfg.D, cfg.K, lengths, seed)
    if cfg.K == 0:
        g = rng(seed + 11)
        width = (2 if cfg.bidirectional else 1) * cfg.H
        dy = g.standard_normal((cfg.T, cfg.B, width)).astype(np.float32)
        dy[batch.mask == 0] = 0.0
        batch.dy_top = dy
    params = stack_params(cfg.L, cfg.D, cfg.H, cfg.K, cfg.bidirectional)
    return cfg, params, batch


def random_small_case(seed: int, T: int, B: int, D: int, H: int,
                      lengths: Optional[np.ndarray] = None, state_scale: float = 0.5):
    """Small random single-layer case with nonzero h0/c0/dy/dhT/dcT (tests)."""
    g = rng(seed)
    if lengths is None:
        lengths = g.integers(1, T + 1, size=B).astype(np.int32)
        lengths[0] = T
    x = g.standard_normal((T, B, D)).astype(np.float32)
    mask = mask_from_lengths(T, lengths)
    W = (0.5 * g.standard_normal((D, 4 * H))).astype(np.float32)
    R = (0.5 * g.standard_normal((H, 4 * H))).astype(np.float32)
    b = (0.5 * g.standard_normal(4 * H)).astype(np.float32)
    h0 = (state_scale * g.standard_normal((B, H))).astype(np.float32)
    c0 = (state_scale * g.standard_normal((B, H))).astype(np.float32)
    dy = g.standard_normal((T, B, H)).astype(np.float32)
    dhT = g.standard_normal((B, H)).astype(np.float32)
    dcT = g.standard_normal((B, H)).astype(np.float32)
    return dict(x=x, mask=mask, W=W, R=R, b=b, h0=h0, c0=c0, dy=dy, dhT=dhT,
                dcT=dcT, lengths=lengths)


# ----------------------------------------------------------------------------
# NEXT-1: a synthetic labelling task with a learnable answer, for the
# convergence study of the paper's K-step parameter averaging (§4.1).
# ----------------------------------------------------------------------------
ECHO_SYMBOLS = 10   # input alphabet 1..V
ECHO_DELAY = 3      # label at frame t = input symbol at frame t - k ("delayed echo, k=3")


def echo_batch(T: int, B: int, D: int, seed: int, V: int = ECHO_SYMBOLS, delay: int = ECHO_DELAY,
               min_len: Optional[int] = None) -> Batch:
    """Delayed echo: symbol s_t ~ U{1..V} per frame, x_t = one-hot(s_t) in dims 0..V-1 plus
    N(0, 0.1^2) noise in the other D-V dims; label_t = s_{t-delay} (0 = "blank" for t < delay);
    K = V + 1 classes.  Variable lengths U{min_len..T} (one sequence of length T), trailing
    padding (x = 0, label 0)."""
    assert D > V
    g = rng(seed)
    lo = min_len if min_len is not None else max(delay + 1, T // 2)
    lengths = g.integers(lo, T + 1, size=B).astype(np.int32)
    lengths[g.integers(0, B)] = T
    mask = mask_from_lengths(T, lengths)
    s = g.integers(1, V + 1, size=(T, B)).astype(np.int32)
    x = np.zeros((T, B, D), np.float32)
    x[..., V:] = (0.1 * g.standard_normal((T, B, D - V))).astype(np.float32)
    tt, bb = np.meshgrid(np.arange(T), np.arange(B), indexing="ij")
    x[tt, bb, s - 1] = 1.0
    labels = np.zeros((T, B), np.int32)
    labels[delay:] = s[:-delay]
    x[mask == 0] = 0.0
    labels[mask == 0] = 0
    return Batch(x=x, mask=mask, labels=labels, lengths=lengths)
