"""Shared test utilities (vectorised restatements of the oracle's init hashes,
checked against oracle/liboracle.so in tests/test_oracle.py)."""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64_np(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def weight_rows(seed: int, table_id: int, rows, dim: int) -> np.ndarray:
    """W_t[rows, :] of the counter-hash init (oracle.c orc_weight_init)."""
    rows = np.asarray(rows, dtype=np.uint64)
    s0 = splitmix64_np(np.uint64(seed))
    key = (np.uint64(table_id) << np.uint64(40)) | (rows[:, None] << np.uint64(10)) | np.arange(
        dim, dtype=np.uint64)[None, :]
    h = splitmix64_np(s0 ^ key)
    k = (h >> np.uint64(54)).astype(np.int64) - 512
    return (k.astype(np.float32) * np.float32(2.0 ** -12)).astype(np.float32)


def grad_grid(seed: int, B: int, ncols: int) -> np.ndarray:
    """G[b, col] of oracle.c orc_grad_init."""
    s = splitmix64_np(np.uint64(seed) ^ np.uint64(0x5EEDF00D5EEDF00D))
    key = (np.arange(B, dtype=np.uint64)[:, None] << np.uint64(20)) | np.arange(ncols, dtype=np.uint64)[None, :]
    h = splitmix64_np(s ^ key)
    k = (h >> np.uint64(54)).astype(np.int64) - 512
    return (k.astype(np.float32) * np.float32(2.0 ** -12)).astype(np.float32)


def to_oracle_tables(tables):
    from oracle import Table

    return [Table(t.id, t.dim, t.hash_size, t.pooling_mean, t.access_ratio, t.bytes_per_param) for t in tables]


def bag_ids(offsets) -> np.ndarray:
    off = np.asarray(offsets, dtype=np.int64)
    return np.repeat(np.arange(len(off) - 1, dtype=np.int32), np.diff(off))


def fp_close(got, ref, rtol=1e-5, atol=1e-7, scale=None):
    """|got - ref| <= rtol*max(|ref|, scale) + atol elementwise.

    `scale` carries the magnitude of the terms that produced ref (e.g. the old
    weight of an Adagrad update W_old - u): when they cancel, ref alone
    understates the fp32 rounding the result legitimately carries."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(got - ref)
    mag = np.abs(ref) if scale is None else np.maximum(np.abs(ref), np.abs(np.asarray(scale, dtype=np.float64)))
    bound = rtol * mag + atol
    ok = err <= bound
    return bool(ok.all()), float((err / np.maximum(bound, 1e-300)).max()) if err.size else 0.0
