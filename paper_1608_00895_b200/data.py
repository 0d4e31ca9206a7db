"""Chunked data pipeline (§4): the step before the
hot path.

Sequences are cut into (possibly overlapping) chunks of constant length C with step S
(starts {0, S, 2S, ...} ∩ [0, L), final chunk zero-padded), the chunks of an
epoch are shuffled by a seed and packed greedily into batches of B chunks (the
paper's CHiME setup uses C = 250, B = 81).  The corpus lives in HBM as one
[frames, D] fp32 array plus int32 frame labels (DeviceCorpus); each batch's x [C, B, D],
mask [C, B] and labels [C, B] are gathered on the device by blstm_gather_chunks, so a step
moves only its B-entry chunk table host -> device.

Valid-frame accounting: with S < C a frame is trained on once per chunk covering it;
chunk_frames() counts frames as the batches see them (the metric's unit), corpus_frames()
counts each frame once.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import numpy as np


@dataclass(frozen=True)
class Chunk:
    seq: int
    start: int
    valid_len: int


def chunk_sequences(lengths: Sequence[int], C: int, S: int) -> List[Chunk]:
    """Chunks of every sequence, in sequence order."""
    if not (1 <= S <= C):
        raise ValueError("chunk step must satisfy 1 <= S <= C")
    if len(lengths) == 0:
        raise ValueError("empty dataset")
    out = []
    for s, L in enumerate(lengths):
        starts = np.arange(0, int(L), S)
        out.extend(Chunk(s, int(a), int(min(C, L - a))) for a in starts)
    return out


def make_batches(chunks: List[Chunk], B: int, seed: int) -> List[List[Chunk]]:
    """Seeded shuffle, then greedy fill: every batch has B chunks except possibly the last."""
    if B < 1:
        raise ValueError("B >= 1")
    order = np.random.Generator(np.random.PCG64(seed)).permutation(len(chunks))
    return [[chunks[i] for i in order[k:k + B]] for k in range(0, len(chunks), B)]


def chunk_frames(batches) -> int:
    return sum(c.valid_len for b in batches for c in b)


class DeviceCorpus:
    """A corpus resident in device memory: frames [F, D] fp32, labels [F] int32 (or None),
    sequence offsets; batches gathered by blstm_gather_chunks."""

    def __init__(self, seqs_x: Sequence[np.ndarray], seqs_labels, device):
        import torch
        self.torch = torch
        self.lengths = np.array([len(x) for x in seqs_x], np.int64)
        self.offset = np.concatenate([[0], np.cumsum(self.lengths)]).astype(np.int64)
        self.D = int(seqs_x[0].shape[1])
        self.frames = torch.tensor(np.concatenate(seqs_x).astype(np.float32), device=device)
        self.labels = (torch.tensor(np.concatenate(seqs_labels).astype(np.int32), device=device)
                       if seqs_labels is not None else None)
        self.device = device

    def corpus_frames(self) -> int:
        return int(self.lengths.sum())

    def gather(self, batch: List[Chunk], T: int, x, mask, labels=None, stream=None):
        """Fill x [T, B, D], mask [T, B] (and labels [T, B]) for the chunks of `batch` (B = its
        width; columns past len(batch) become padding)."""
        from . import blstm
        B = x.shape[1]
        start = np.zeros(B, np.int64)
        n = np.zeros(B, np.int32)
        for b, c in enumerate(batch):
            if c.valid_len > T:
                raise ValueError("chunk longer than T")
            start[b] = self.offset[c.seq] + c.start
            n[b] = c.valid_len
        t = self.torch
        st = t.tensor(start, device=self.device)
        nl = t.tensor(n, device=self.device)
        blstm.blstm_gather_chunks(self.frames, self.labels, self.D, st, nl, B, T, x, mask, labels, stream)

    def plan_epoch(self, batches: List[List[Chunk]], B: int, T: int):
        """Upload the chunk tables of a whole epoch once (int64 starts / int32 lengths [n, B]);
        gather_planned(k, ...) then moves no host data per step."""
        t = self.torch
        n = len(batches)
        start = np.zeros((n, B), np.int64)
        ln = np.zeros((n, B), np.int32)
        for k, batch in enumerate(batches):
            for b, c in enumerate(batch):
                if c.valid_len > T:
                    raise ValueError("chunk longer than T")
                start[k, b] = self.offset[c.seq] + c.start
                ln[k, b] = c.valid_len
        self.plan = (t.tensor(start, device=self.device), t.tensor(ln, device=self.device), B, T)
        return n

    def gather_planned(self, k: int, x, mask, labels=None, stream=None):
        from . import blstm
        start, ln, B, T = self.plan
        blstm.blstm_gather_chunks(self.frames, self.labels, self.D, start[k], ln[k], B, T, x, mask, labels, stream)
