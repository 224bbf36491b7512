"""Shared builders for parity tests (synthetic, seeded inputs)."""
from __future__ import annotations

import numpy as np


def paged_layout(seq_lens, page=64, extra_pages=3, seed=0):
    """Random page assignment: returns (block_table [B,max_pages] int32, num_pages)."""
    rng = np.random.default_rng(seed)
    need = [max(0, (L + page - 1) // page) for L in seq_lens]
    max_pages = max(1, max(need))
    num_pages = sum(need) + extra_pages
    perm = rng.permutation(num_pages).astype(np.int32)
    bt = np.zeros((len(seq_lens), max_pages), np.int32)
    k = 0
    for b, n in enumerate(need):
        bt[b, :n] = perm[k:k + n]
        k += n
    return bt, num_pages


def rel_err(got, ref):
    """max |got-ref| normalised by max |ref| (the stated tolerance metric)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-12))


def rel_fro(got, ref):
    """normwise relative error ||got-ref||_2 / ||ref||_2 (accuracy of a format)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))


def record(name, **vals):
    """Append a measured parity figure to $PARITY_LOG (JSON lines) when set, so
    the errors behind DESIGN.md's parity table come from the GPU run itself."""
    import json
    import os

    path = os.environ.get("PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": name, **{k: float(v) for k, v in vals.items()}}) + "\n")
