"""TEST INFRASTRUCTURE ONLY — ctypes views of the CPU oracle and of the
reference compiled in place.

* ``Oracle``  — ``oracle/liboracle.so``: plain-C restatement of the reference
  generator/planners (autoshard/rng.hpp, tables.hpp, planners.hpp) plus the
  embedding-bag arithmetic the reference lacks (see oracle/oracle.h).
* ``Ref``     — ``oracle/_ref/libref.so``: the UNMODIFIED reference headers
  (/root/reference/proj/include) behind a C shim (oracle/ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this package. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref.so")


class TableC(C.Structure):
    """Layout shared by orc_table, as_table_spec and the ref shim."""

    _fields_ = [
        ("id", C.c_int32),
        ("dim", C.c_int32),
        ("hash_size", C.c_int64),
        ("pooling_mean", C.c_double),
        ("access_ratio", C.c_double),
        ("bytes_per_param", C.c_int32),
        ("_pad", C.c_int32),
    ]


class GenCfgC(C.Structure):
    _fields_ = [
        ("hash_size_min", C.c_double),
        ("hash_size_max", C.c_double),
        ("pooling_mean_target", C.c_double),
        ("pooling_shape", C.c_double),
        ("pooling_cap", C.c_double),
        ("dim_choices", C.POINTER(C.c_int32)),
        ("n_dim_choices", C.c_int32),
        ("access_ratio_min", C.c_double),
        ("access_ratio_max", C.c_double),
        ("bytes_per_param", C.c_int32),
    ]


@dataclass
class Table:
    id: int
    dim: int
    hash_size: int
    pooling_mean: float
    access_ratio: float
    bytes_per_param: int = 2


def tables_to_c(tables):
    arr = (TableC * max(1, len(tables)))()
    for i, t in enumerate(tables):
        arr[i] = TableC(t.id, t.dim, t.hash_size, t.pooling_mean, t.access_ratio, t.bytes_per_param, 0)
    return arr


def tables_from_c(arr, n):
    return [Table(arr[i].id, arr[i].dim, arr[i].hash_size, arr[i].pooling_mean,
                  arr[i].access_ratio, arr[i].bytes_per_param) for i in range(n)]


GEN_DEFAULTS = dict(hash_size_min=1e3, hash_size_max=1e7, pooling_mean_target=15.0,
                    pooling_shape=2.0, pooling_cap=193.0, dim_choices=(16, 32),
                    access_ratio_min=1e-3, access_ratio_max=1.0, bytes_per_param=2)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"oracle library missing: {path} (run __graft_entry__.build())")
        L = self.lib = C.CDLL(path)
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_fnv1a64.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64]
        L.orc_generate_pool.argtypes = [C.c_uint64, C.c_int, C.POINTER(GenCfgC), C.POINTER(TableC)]
        L.orc_generate_stream.argtypes = [C.c_uint64, C.POINTER(TableC), C.c_int64, C.c_double,
                                          C.POINTER(C.POINTER(C.c_int64)),
                                          C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.c_int64)]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_fingerprint_pool.restype = C.c_uint64
        L.orc_fingerprint_pool.argtypes = [C.POINTER(TableC), C.c_int]
        L.orc_fingerprint_task.restype = C.c_uint64
        L.orc_fingerprint_task.argtypes = [C.POINTER(TableC), C.c_int, C.c_int, C.POINTER(C.c_int64)]
        L.orc_greedy_shard.argtypes = [C.POINTER(TableC), C.c_int, C.c_int, C.POINTER(C.c_int64),
                                       C.c_int, C.POINTER(C.c_int)]
        L.orc_random_shard.argtypes = [C.POINTER(TableC), C.c_int, C.c_int, C.POINTER(C.c_int64),
                                       C.c_uint64, C.POINTER(C.c_int)]
        L.orc_degree_of_balance.restype = C.c_double
        L.orc_degree_of_balance.argtypes = [C.POINTER(C.c_double), C.c_int]
        L.orc_weight_init.restype = C.c_float
        L.orc_weight_init.argtypes = [C.c_uint64, C.c_int32, C.c_int64, C.c_int32]
        L.orc_fill_weights.argtypes = [C.c_uint64, C.c_int32, C.c_int64, C.c_int32, C.POINTER(C.c_float)]
        L.orc_grad_init.restype = C.c_float
        L.orc_grad_init.argtypes = [C.c_uint64, C.c_int64, C.c_int64]
        L.orc_emb_forward_f64.argtypes = [C.c_int, C.POINTER(TableC), C.c_int64,
                                          C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                          C.POINTER(C.c_void_p), C.c_uint64, C.POINTER(C.c_double)]
        L.orc_emb_forward_f64_rows.argtypes = [C.c_int, C.POINTER(TableC), C.c_int64, C.c_int64, C.c_int64,
                                               C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                               C.POINTER(C.c_void_p), C.c_uint64, C.POINTER(C.c_double)]
        L.orc_emb_backward_adagrad_f64.argtypes = [
            C.POINTER(TableC), C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
            C.POINTER(C.c_float), C.c_int64, C.c_int64, C.POINTER(C.c_float), C.POINTER(C.c_float),
            C.c_uint64, C.c_double, C.c_double, C.POINTER(C.c_int64),
            C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.POINTER(C.c_int64)),
            C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.POINTER(C.c_double))]
        L.orc_cpu_step_f32.restype = C.c_int
        L.orc_cpu_step_f32.argtypes = [C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.c_int64,
                                       C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_float),
                                       C.c_float, C.c_float, C.c_int]

    # -- generator / planners ------------------------------------------------
    def generate_pool(self, seed, n, **cfg):
        c = dict(GEN_DEFAULTS)
        c.update(cfg)
        dims = (C.c_int32 * len(c["dim_choices"]))(*c["dim_choices"])
        g = GenCfgC(c["hash_size_min"], c["hash_size_max"], c["pooling_mean_target"],
                    c["pooling_shape"], c["pooling_cap"], dims, len(c["dim_choices"]),
                    c["access_ratio_min"], c["access_ratio_max"], c["bytes_per_param"])
        out = (TableC * n)()
        rc = self.lib.orc_generate_pool(seed, n, C.byref(g), out)
        if rc:
            raise ValueError(f"orc_generate_pool rc={rc}")
        return tables_from_c(out, n)

    def generate_stream(self, seed, table, batch, zipf=1.05):
        """(offsets int64[B+1], indices int64[L]) for one table."""
        tc = tables_to_c([table])
        po, pi, n = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.c_int64()
        rc = self.lib.orc_generate_stream(seed, tc, batch, zipf, C.byref(po), C.byref(pi), C.byref(n))
        if rc:
            raise ValueError(f"orc_generate_stream rc={rc}")
        off = np.ctypeslib.as_array(po, shape=(batch + 1,)).copy()
        idx = np.ctypeslib.as_array(pi, shape=(max(n.value, 1),))[: n.value].copy()
        self.lib.orc_free(po)
        self.lib.orc_free(pi)
        return off, idx

    def generate_workload(self, seed, tables, batch, zipf=1.05):
        return {t.id: self.generate_stream(seed, t, batch, zipf) for t in sorted(tables, key=lambda t: t.id)}

    def fnv(self, data: bytes, h=0xcbf29ce484222325):
        return self.lib.orc_fnv1a64(data, len(data), h)

    def fingerprint_pool(self, tables):
        return self.lib.orc_fingerprint_pool(tables_to_c(tables), len(tables))

    def fingerprint_task(self, tables, budgets):
        b = np.asarray(budgets, dtype=np.int64)
        return self.lib.orc_fingerprint_task(tables_to_c(tables), len(tables), len(b), _p(b, C.c_int64))

    def greedy_shard(self, tables, budgets, kind):
        b = np.asarray(budgets, dtype=np.int64)
        out = (C.c_int * max(1, len(tables)))()
        rc = self.lib.orc_greedy_shard(tables_to_c(tables), len(tables), len(b), _p(b, C.c_int64), kind, out)
        if rc:
            raise ValueError(f"orc_greedy_shard rc={rc}")
        return list(out)[: len(tables)]

    def random_shard(self, tables, budgets, seed):
        b = np.asarray(budgets, dtype=np.int64)
        out = (C.c_int * max(1, len(tables)))()
        rc = self.lib.orc_random_shard(tables_to_c(tables), len(tables), len(b), _p(b, C.c_int64), seed, out)
        if rc:
            raise ValueError(f"orc_random_shard rc={rc}")
        return list(out)[: len(tables)]

    def degree_of_balance(self, costs):
        c = np.asarray(costs, dtype=np.float64)
        return self.lib.orc_degree_of_balance(_p(c, C.c_double), len(c))

    # -- arithmetic ---------------------------------------------------------
    def weight_init(self, seed, table_id, row, d):
        return self.lib.orc_weight_init(seed, table_id, row, d)

    def dense_weights(self, seed, table):
        """Dense fp32 init of one (small) table, via the oracle hash."""
        W = np.empty((table.hash_size, table.dim), dtype=np.float32)
        f = self.lib.orc_weight_init
        for r in range(table.hash_size):
            for d in range(table.dim):
                W[r, d] = f(seed, table.id, r, d)
        return W

    def fill_weights(self, seed, table, out=None):
        """Dense [hash, dim] fp32 init of one table (OpenMP C)."""
        if out is None:
            out = np.empty((table.hash_size, table.dim), dtype=np.float32)
        self.lib.orc_fill_weights(seed, table.id, table.hash_size, table.dim, _p(out, C.c_float))
        return out

    def grad_init(self, seed, B, ncols):
        f = self.lib.orc_grad_init
        return np.array([[f(seed, b, c) for c in range(ncols)] for b in range(B)], dtype=np.float32)

    def forward_f64(self, tables, B, streams, wseed=0, dense=None, rows=None):
        """streams: list of (offsets, indices) in `tables` order. Returns [B, sum(dim)] fp64
        (rows=(b0, b1): only those batch rows, [b1 - b0, sum(dim)]; OpenMP)."""
        T = len(tables)
        offs = [np.ascontiguousarray(s[0], dtype=np.int64) for s in streams]
        idxs = [np.ascontiguousarray(s[1], dtype=np.int64) for s in streams]
        po = (C.c_void_p * T)(*[o.ctypes.data for o in offs])
        pi = (C.c_void_p * T)(*[i.ctypes.data for i in idxs])
        pw = None
        if dense is not None:
            dense = [np.ascontiguousarray(w, dtype=np.float32) for w in dense]
            pw = (C.c_void_p * T)(*[w.ctypes.data for w in dense])
        b0, b1 = rows if rows is not None else (0, B)
        out = np.empty((b1 - b0, sum(t.dim for t in tables)), dtype=np.float64)
        self.lib.orc_emb_forward_f64_rows(T, tables_to_c(tables), B, b0, b1, po, pi, pw, wseed,
                                          _p(out, C.c_double))
        return out

    def backward_adagrad_f64(self, table, B, offsets, indices, grad, col0, lr, eps,
                             wseed=0, W=None, M=None):
        """Returns dict(rows, counts, w, m). W/M dense fp32 arrays updated in place if given."""
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        indices = np.ascontiguousarray(indices, dtype=np.int64)
        grad = np.ascontiguousarray(grad, dtype=np.float32)
        nu = C.c_int64()
        pr, pc = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
        pw, pm = C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
        self.lib.orc_emb_backward_adagrad_f64(
            tables_to_c([table]), B, _p(offsets, C.c_int64), _p(indices, C.c_int64),
            _p(grad, C.c_float), grad.shape[1], col0,
            _p(W, C.c_float) if W is not None else None, _p(M, C.c_float) if M is not None else None,
            wseed, lr, eps, C.byref(nu), C.byref(pr), C.byref(pc), C.byref(pw), C.byref(pm))
        U = nu.value
        D = table.dim

        def take(p, shape, dt):
            if U == 0:
                self.lib.orc_free(p)
                return np.zeros(shape, dtype=dt)
            a = np.ctypeslib.as_array(p, shape=shape).copy()
            self.lib.orc_free(p)
            return a

        return dict(rows=take(pr, (U,), np.int64), counts=take(pc, (U,), np.int64),
                    w=take(pw, (U, D), np.float64), m=take(pm, (U,), np.float64))

    def cpu_step_f32(self, dims, hashes, B, streams, W_all, M_all, out, lr, eps, n_threads=0):
        T = len(dims)
        d = np.asarray(dims, dtype=np.int32)
        h = np.asarray(hashes, dtype=np.int64)
        offs = [np.ascontiguousarray(s[0], dtype=np.int64) for s in streams]
        idxs = [np.ascontiguousarray(s[1], dtype=np.int64) for s in streams]
        po = (C.c_void_p * T)(*[o.ctypes.data for o in offs])
        pi = (C.c_void_p * T)(*[i.ctypes.data for i in idxs])
        return self.lib.orc_cpu_step_f32(T, _p(d, C.c_int32), _p(h, C.c_int64), B, po, pi,
                                         _p(W_all, C.c_float), _p(M_all, C.c_float), _p(out, C.c_float),
                                         lr, eps, n_threads)


class Ref:
    """The unmodified reference, compiled in place (oracle/_ref/libref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"reference build missing: {path}")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_generate_pool.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_double, C.POINTER(C.c_int), C.c_int,
                                        C.c_double, C.c_double, C.c_int, C.POINTER(TableC)]
        L.ref_generate_workload.argtypes = [C.c_uint64, C.POINTER(TableC), C.c_int, C.c_int64,
                                            C.c_double, C.POINTER(C.c_void_p)]
        L.ref_workload_table.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int),
                                         C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.c_int64),
                                         C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.c_int64)]
        L.ref_workload_free.argtypes = [C.c_void_p]
        L.ref_fingerprint_pool.restype = C.c_uint64
        L.ref_fingerprint_pool.argtypes = [C.POINTER(TableC), C.c_int]
        L.ref_fingerprint_task.restype = C.c_uint64
        L.ref_fingerprint_task.argtypes = [C.POINTER(TableC), C.c_int, C.c_int, C.POINTER(C.c_int64)]
        L.ref_serialized_hash.argtypes = [C.POINTER(TableC), C.c_int, C.c_void_p,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.ref_save_workload_file.argtypes = [C.c_char_p, C.c_void_p]
        L.ref_load_workload_file.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_greedy_shard.argtypes = [C.POINTER(TableC), C.c_int, C.c_int, C.POINTER(C.c_int64),
                                       C.c_int, C.POINTER(C.c_int)]
        L.ref_random_shard.argtypes = [C.POINTER(TableC), C.c_int, C.c_int, C.POINTER(C.c_int64),
                                       C.c_uint64, C.POINTER(C.c_int)]
        L.ref_degree_of_balance.argtypes = [C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double)]
        L.ref_measure_plan.argtypes = [C.POINTER(TableC), C.c_int, C.c_int, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int), C.c_void_p, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_uint64, C.POINTER(C.c_double)]

    def _chk(self, rc):
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def generate_pool(self, seed, n, **cfg):
        c = dict(GEN_DEFAULTS)
        c.update(cfg)
        dims = (C.c_int * len(c["dim_choices"]))(*c["dim_choices"])
        out = (TableC * n)()
        self._chk(self.lib.ref_generate_pool(seed, n, c["hash_size_min"], c["hash_size_max"],
                                             c["pooling_mean_target"], c["pooling_shape"],
                                             c["pooling_cap"], dims, len(c["dim_choices"]),
                                             c["access_ratio_min"], c["access_ratio_max"],
                                             c["bytes_per_param"], out))
        return tables_from_c(out, n)

    def generate_workload(self, seed, tables, batch, zipf=1.05):
        """Returns (handle, {table_id: (offsets, indices)}); free with free_workload."""
        h = C.c_void_p()
        self._chk(self.lib.ref_generate_workload(seed, tables_to_c(tables), len(tables), batch, zipf,
                                                 C.byref(h)))
        out = {}
        for i in range(len(tables)):
            tid = C.c_int()
            po, pi = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
            no, ni = C.c_int64(), C.c_int64()
            self.lib.ref_workload_table(h, i, C.byref(tid), C.byref(po), C.byref(no), C.byref(pi), C.byref(ni))
            off = np.ctypeslib.as_array(po, shape=(no.value,)).copy()
            idx = (np.ctypeslib.as_array(pi, shape=(ni.value,)).copy() if ni.value
                   else np.zeros(0, dtype=np.int64))
            out[tid.value] = (off, idx)
        return h, out

    def free_workload(self, h):
        self.lib.ref_workload_free(h)

    def serialized_hash(self, pool, handle):
        hsh, nb = C.c_uint64(), C.c_uint64()
        self._chk(self.lib.ref_serialized_hash(tables_to_c(pool), len(pool), handle, C.byref(hsh), C.byref(nb)))
        return hsh.value, nb.value

    def fingerprint_pool(self, tables):
        return self.lib.ref_fingerprint_pool(tables_to_c(tables), len(tables))

    def fingerprint_task(self, tables, budgets):
        b = np.asarray(budgets, dtype=np.int64)
        return self.lib.ref_fingerprint_task(tables_to_c(tables), len(tables), len(b), _p(b, C.c_int64))

    def greedy_shard(self, tables, budgets, kind):
        b = np.asarray(budgets, dtype=np.int64)
        out = (C.c_int * max(1, len(tables)))()
        self._chk(self.lib.ref_greedy_shard(tables_to_c(tables), len(tables), len(b), _p(b, C.c_int64), kind, out))
        return list(out)[: len(tables)]

    def random_shard(self, tables, budgets, seed):
        b = np.asarray(budgets, dtype=np.int64)
        out = (C.c_int * max(1, len(tables)))()
        self._chk(self.lib.ref_random_shard(tables_to_c(tables), len(tables), len(b), _p(b, C.c_int64), seed, out))
        return list(out)[: len(tables)]

    def measure_plan(self, tables, budgets, assignment, handle, warmup=5, measure=10, trim=2,
                     exact=False, seed=0):
        b = np.asarray(budgets, dtype=np.int64)
        a = (C.c_int * len(assignment))(*assignment)
        out = (C.c_double * len(b))()
        self._chk(self.lib.ref_measure_plan(tables_to_c(tables), len(tables), len(b), _p(b, C.c_int64),
                                            a, handle, warmup, measure, trim, int(exact), seed, out))
        return list(out)


def stream_hash(fnv, streams_in_id_order):
    """SURVEY.md §8c stream hash: fnv1a64 seeded with fnv1a64("wl") over each
    table's int64 offsets then indices, tables ascending by id."""
    h = fnv(b"wl")
    for off, idx in streams_in_id_order:
        h = fnv(np.ascontiguousarray(off, dtype=np.int64).tobytes(), h)
        h = fnv(np.ascontiguousarray(idx, dtype=np.int64).tobytes(), h)
    return h
