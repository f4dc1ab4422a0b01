"""The CPU oracle is pinned before it is trusted (CPU only):
* against the golden vectors generated from the reference compiled in place
  (tests/golden/golden.json, SURVEY.md §8c hashes);
* against the live reference build (oracle/_ref) on randomized configs, when present;
* its embedding-bag arithmetic (absent from the reference) against torch's
  CPU embedding_bag (forward) and an independent numpy restatement (backward).
"""
import json
import os

import numpy as np
import pytest

from helpers import bag_ids, grad_grid, weight_rows

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def plan_str(a):
    return "".join(map(str, a))


def test_oracle_cfg1_golden(oracle):
    from oracle import stream_hash

    pool = oracle.generate_pool(0, 10, dim_choices=(64,), pooling_mean_target=20.0)
    assert f"{oracle.fingerprint_pool(pool):016x}" == GOLD["cfg1"]["fingerprint_pool"] == "666597d9931b028c"
    w = oracle.generate_workload(0, pool, 512)
    assert f"{stream_hash(oracle.fnv, [w[t.id] for t in pool]):016x}" == GOLD["cfg1"]["stream_hash"]
    assert sum(len(w[t.id][1]) for t in pool) == GOLD["cfg1"]["lookups"] == 97148
    assert sum(len(np.unique(w[t.id][1])) for t in pool) == GOLD["cfg1"]["unique_rows"] == 12473
    assert w[pool[0].id][0][:65].tolist() == GOLD["cfg1"]["table0_offsets_head"]
    assert w[pool[0].id][1][:64].tolist() == GOLD["cfg1"]["table0_indices_head"]
    b = GOLD["cfg1"]["budget"]
    for i, k in enumerate(["size", "dim", "lookup"]):
        assert plan_str(oracle.greedy_shard(pool, b, i)) == GOLD["cfg1"]["plans"][k]
    assert plan_str(oracle.random_shard(pool, b, 0)) == GOLD["cfg1"]["plans"]["random0"]
    assert f"{oracle.fingerprint_task(pool, b):016x}" == GOLD["cfg1"]["fingerprint_task"]


def test_oracle_cfg2_golden(oracle):
    from oracle import Table, stream_hash

    pool = oracle.generate_pool(0, 856)
    assert f"{oracle.fingerprint_pool(pool):016x}" == GOLD["pool856_fingerprint"]
    p2 = [Table(t.id, 128, t.hash_size, t.pooling_mean, t.access_ratio, t.bytes_per_param) for t in pool[:50]]
    b = GOLD["cfg2"]["budget"]
    for i, k in enumerate(["size", "dim", "lookup"]):
        assert plan_str(oracle.greedy_shard(p2, b, i)) == GOLD["cfg2"]["plans"][k]
    assert plan_str(oracle.random_shard(p2, b, 0)) == GOLD["cfg2"]["plans"]["random0"]
    w = oracle.generate_workload(0, p2, 65536)
    assert f"{stream_hash(oracle.fnv, [w[t.id] for t in p2]):016x}" == GOLD["cfg2"]["stream_hash"] == "76a2fdd3d7b504ca"


def test_oracle_spec_greedy_fixture(oracle):
    from oracle import Table

    spec = [Table(i, 1, 10, float(c), 1.0, 1) for i, c in enumerate([4, 3, 3, 2, 2])]
    a = oracle.greedy_shard(spec, [10 ** 9, 10 ** 9], 2)
    assert a == GOLD["spec_greedy"]["assignment"]
    loads = [sum(c for c, k in zip([4, 3, 3, 2, 2], a) if k == s) for s in range(2)]
    assert sorted(loads) == [6, 8]


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_oracle_matches_reference_build(oracle, ref, seed):
    rng = np.random.default_rng(seed)
    cfg = dict(hash_size_min=float(rng.choice([1, 10, 1000])), hash_size_max=float(rng.choice([5e3, 1e5])),
               pooling_mean_target=float(rng.choice([0.0, 3.0, 30.0])), dim_choices=(16, 64, 128),
               access_ratio_min=float(rng.choice([1e-3, 0.5])))
    n = int(rng.integers(1, 20))
    po = oracle.generate_pool(seed, n, **cfg)
    pr = ref.generate_pool(seed, n, **cfg)
    assert po == pr
    B = int(rng.integers(1, 300))
    z = float(rng.choice([1.05, 0.3, 2.0]))
    wo = oracle.generate_workload(seed + 7, po, B, z)
    h, wr = ref.generate_workload(seed + 7, pr, B, z)
    ref.free_workload(h)
    for t in po:
        assert np.array_equal(wo[t.id][0], wr[t.id][0]) and np.array_equal(wo[t.id][1], wr[t.id][1])
    budget = [sum(t.dim * t.hash_size * t.bytes_per_param for t in po)] * 3
    for kind in range(3):
        assert oracle.greedy_shard(po, budget, kind) == ref.greedy_shard(pr, budget, kind)
    assert oracle.random_shard(po, budget, seed) == ref.random_shard(pr, budget, seed)
    tight = [max(t.dim * t.hash_size * t.bytes_per_param for t in po)] * 4
    if sum(tight) >= sum(t.dim * t.hash_size * t.bytes_per_param for t in po):
        assert oracle.greedy_shard(po, tight, 2) == ref.greedy_shard(pr, tight, 2)
        assert oracle.random_shard(po, tight, 5) == ref.random_shard(pr, tight, 5)


def test_oracle_canonical_serialization(ref):
    pool = ref.generate_pool(0, 856)
    h, _ = ref.generate_workload(0, pool[:40], 4096)
    hh, nb = ref.serialized_hash(pool, h)
    ref.free_workload(h)
    assert f"{hh:016x}" == GOLD["canonical"]["hash"] == "9c582e4bb6abc304" and nb == 13452245


def test_oracle_forward_matches_torch_embedding_bag(oracle):
    torch = pytest.importorskip("torch")
    pool = oracle.generate_pool(3, 4, dim_choices=(8, 16), hash_size_max=3e3, pooling_mean_target=12.0)
    B = 50
    w = oracle.generate_workload(1, pool, B)
    st = [w[t.id] for t in pool]
    out = oracle.forward_f64(pool, B, st, wseed=5)
    col = 0
    for t, (off, idx) in zip(pool, st):
        W = torch.from_numpy(weight_rows(5, t.id, np.arange(t.hash_size), t.dim).astype(np.float64))
        ref = torch.nn.functional.embedding_bag(torch.from_numpy(idx), W, torch.from_numpy(off[:-1]), mode="sum")
        assert np.array_equal(out[:, col:col + t.dim], ref.numpy())
        col += t.dim


def test_oracle_backward_matches_numpy(oracle):
    pool = oracle.generate_pool(4, 3, dim_choices=(4, 12), hash_size_min=50.0, hash_size_max=500.0, pooling_mean_target=9.0)
    B, lr, eps = 40, 0.1, 1e-6
    w = oracle.generate_workload(2, pool, B)
    SD = sum(t.dim for t in pool)
    G = grad_grid(3, B, SD)
    col = 0
    for t in pool:
        off, idx = w[t.id]
        r = oracle.backward_adagrad_f64(t, B, off, idx, G, col, lr, eps, wseed=6)
        rows, counts = np.unique(idx, return_counts=True)
        assert np.array_equal(r["rows"], rows) and np.array_equal(r["counts"], counts)
        g = np.zeros((t.hash_size, t.dim))
        np.add.at(g, idx, G[bag_ids(off), col:col + t.dim].astype(np.float64))
        g = g[rows]
        m = (g * g).sum(1) / t.dim
        W0 = weight_rows(6, t.id, rows, t.dim).astype(np.float64)
        want = W0 - (lr / (np.sqrt(m) + eps))[:, None] * g
        assert np.allclose(r["m"], m, rtol=1e-12) and np.allclose(r["w"], want, rtol=1e-12, atol=1e-15)
        col += t.dim


def test_oracle_init_hash_vectorised_agrees(oracle):
    from oracle import Table

    t = Table(7, 12, 300, 1.0, 1.0)
    d = oracle.fill_weights(11, t)
    assert np.array_equal(d, weight_rows(11, 7, np.arange(300), 12))
    assert oracle.weight_init(11, 7, 299, 11) == d[299, 11]
    assert np.array_equal(grad_grid(2, 5, 7), oracle.grad_init(2, 5, 7))
    vals = np.unique(d)
    assert vals.min() >= -0.125 and vals.max() < 0.125 and np.all(vals * 4096 == np.round(vals * 4096))


def test_cpu_step_port_matches_f64_oracle(oracle):
    """The fp32 OpenMP port (the timed CPU baseline) computes the same step."""
    pool = oracle.generate_pool(2, 3, dim_choices=(8,), hash_size_min=50.0, hash_size_max=400.0, pooling_mean_target=6.0)
    B, lr, eps, seed = 64, 0.05, 1e-6, 0
    w = oracle.generate_workload(4, pool, B)
    st = [w[t.id] for t in pool]
    W = np.concatenate([weight_rows(seed, t.id, np.arange(t.hash_size), t.dim).ravel() for t in pool])
    M = np.zeros(sum(t.hash_size for t in pool), dtype=np.float32)
    out = np.empty((B, 8 * len(pool)), dtype=np.float32)
    oracle.cpu_step_f32([t.dim for t in pool], [t.hash_size for t in pool], B, st, W, M, out, lr, eps, 2)
    ref = oracle.forward_f64(pool, B, st, wseed=seed)
    assert np.array_equal(out.astype(np.float64), ref)
    off_w = 0
    for k, t in enumerate(pool):
        r = oracle.backward_adagrad_f64(t, B, *st[k], ref.astype(np.float32), 8 * k, lr, eps, wseed=seed)
        Wt = W[off_w:off_w + t.hash_size * t.dim].reshape(t.hash_size, t.dim)
        assert np.allclose(Wt[r["rows"]], r["w"], rtol=1e-5, atol=1e-6)
        off_w += t.hash_size * t.dim


def test_features_numpy_restatement_matches_reference(ref):
    """Pins the numpy extract_features restatement used by the GPU feature
    test against the reference's own extract_features (tables.hpp:344-386)."""
    import ctypes as C

    from test_gpu_parity import _features_np

    pool = ref.generate_pool(0, 6, pooling_mean_target=25.0, hash_size_max=2e4)
    h, w = ref.generate_workload(0, pool, 1024)
    out = (C.c_double * (21 * len(pool)))()
    rc = ref.lib.ref_extract_features(__import__("oracle").tables_to_c(pool), len(pool), h, out)
    ref.free_workload(h)
    assert rc == 0
    got = np.array(list(out)).reshape(len(pool), 21)
    want = np.stack([_features_np(t, w[t.id][1], 1024) for t in pool])
    assert np.array_equal(got, want)
