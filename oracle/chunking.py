"""Oracle of the chunked data pipeline.  TEST INFRASTRUCTURE ONLY:
only tests/, __graft_entry__.smoke() and bench.py's baseline legs may import it.

PAPER.md §4: "an option to chunk sequences into (possibly overlapping) segments of
constant length"; SPEC S:327-330 makes it concrete: chunk starts {0, S, 2S, ...} ∩ [0, L),
chunk size C, step 1 <= S <= C, the final chunk zero-padded, every frame covered by >= 1
chunk.  Plain Python loops, written from those lines; no code shared with the CUDA path.
Pins: tests/test_chunking.py (SPEC's worked examples, coverage, conservation).
"""
import numpy as np


def chunk_starts(L: int, C: int, S: int):
    """[(start, valid_len)] of one sequence of length L."""
    if not (1 <= S <= C):
        raise ValueError("need 1 <= S <= C")
    out = []
    s = 0
    while s < L:
        out.append((s, min(C, L - s)))
        s += S
    return out


def gather_chunks(frames, frame_labels, seq_offset, chunks, T: int):
    """Batch tensors of the chunks [(seq, start, valid_len)] (one column each, in order):
    x [T, B, D] (0 at padding), mask [T, B] uint8, labels [T, B] int32 (0 at padding);
    sequence s occupies frames[seq_offset[s] : seq_offset[s+1]]."""
    B, D = len(chunks), frames.shape[1]
    x = np.zeros((T, B, D), np.float32)
    mask = np.zeros((T, B), np.uint8)
    labels = np.zeros((T, B), np.int32)
    for b, (seq, start, n) in enumerate(chunks):
        for t in range(n):
            f = seq_offset[seq] + start + t
            x[t, b, :] = frames[f, :]
            mask[t, b] = 1
            if frame_labels is not None:
                labels[t, b] = frame_labels[f]
    return x, mask, labels
