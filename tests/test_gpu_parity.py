"""GPU parity of the sm_100a hot path against the CPU oracle, through the C-ABI.

Tolerances:
* forward: BIT-EXACT. Initial weights live on the grid k*2^-12 (|k| <= 512), so
  every partial sum of a bag below 2^12 in magnitude is exact in fp32 whatever
  the summation order; the fp64 oracle must therefore match exactly.
* backward / updated rows: |gpu - ref| <= 1e-5*max(|ref|, |W_old|, |W_old - ref|) + 1e-7
  elementwise (north star: 1e-5 relative fp32; the scale is that of the terms
  of W_old - update, so cancellation to ~0 does not demand more than fp32
  delivers). Momentum: |gpu - ref| <= 1e-5*|ref| + 1e-7. ref in fp64. Gradients
  of rows hit > 2^12 times exceed the exact fp32 grid, so fp32 accumulation
  order matters there; the bound above covers it.
* forward after weights leave the grid (multi-step test): |gpu - ref| <=
  1e-5 * sum_j |W[idx_j]| + 1e-7 (relative to the magnitude of the summands;
  sequential fp32 summation of n terms is bounded by n*2^-24*sum|terms|).
* index handling (bag segmentation, sorted unique rows, counts): bit-exact.
"""
import numpy as np
import pytest

from helpers import bag_ids, fp_close, grad_grid, to_oracle_tables, weight_rows

pytestmark = pytest.mark.gpu

LR, EPS = 0.05, 1e-6


def streams_of(wl, tables):
    return [(wl.find(t.id).offsets, wl.find(t.id).indices) for t in tables]


def run_bwd_check(oracle, shard, tables, streams, grad, seed, B):
    for t, tab in enumerate(tables):
        r = oracle.backward_adagrad_f64(to_oracle_tables([tab])[0], B, *streams[t], grad, shard.cols[t], LR, EPS,
                                        wseed=seed)
        if len(r["rows"]) == 0:
            continue
        w = shard.read_rows(t, r["rows"])
        w_old = weight_rows(seed, tab.id, r["rows"], tab.dim).astype(np.float64)
        scale = np.maximum(np.abs(w_old), np.abs(w_old - r["w"]))
        ok, worst = fp_close(w, r["w"], scale=scale)
        assert ok, f"table {tab.id}: updated rows off by {worst:.3g}x tolerance"
        m = shard.read_momentum(t, r["rows"])
        ok, worst = fp_close(m, r["m"])
        assert ok, f"table {tab.id}: momentum off by {worst:.3g}x tolerance"


def test_cfg1_forward_bitexact_and_segmentation(P, oracle, cuda):
    """BASELINE cfg 1: 10 tables, dim 64, batch 512, mean pooling 20."""
    pool = P.generate_pool(0, 10, P.GeneratorConfig(dim_choices=(64,), pooling_mean_target=20.0))
    B, seed = 512, 3
    wl = P.generate_workload(0, pool, B)
    st = streams_of(wl, pool)
    with P.EmbeddingShard(pool, B, weight_seed=seed) as sh:
        sh.load(st)
        sh.forward()
        got = sh.read_pooled()
        ref = oracle.forward_f64(to_oracle_tables(pool), B, st, wseed=seed)
        assert np.array_equal(got.astype(np.float64), ref)
        # bag segmentation (bit-exact): K4 bag id per lookup, table-major
        assert np.array_equal(sh.read_buffer(P.device.BAG_IDS), np.concatenate([bag_ids(o) for o, _ in st]))
        # device index array = global rows
        row_off = np.cumsum([0] + [t.hash_size for t in pool])[:-1]
        glob = np.concatenate([i + r0 for (_, i), r0 in zip(st, row_off)]).astype(np.int32)
        assert np.array_equal(sh.read_buffer(P.device.GLOBAL_ROWS), glob)
        sh.backward(None, LR, EPS)
        # stable sort by global row with bag ids: bit-exact
        bags = np.concatenate([bag_ids(o) for o, _ in st])
        order = np.argsort(glob, kind="stable")
        assert np.array_equal(sh.read_buffer(P.device.SORTED_ROWS), glob[order])
        assert np.array_equal(sh.read_buffer(P.device.SORTED_BAGS), bags[order])


def test_cfg1_backward_rowwise_adagrad(P, oracle, cuda):
    torch = cuda
    pool = P.generate_pool(0, 10, P.GeneratorConfig(dim_choices=(64,), pooling_mean_target=20.0))
    B, seed = 512, 5
    wl = P.generate_workload(0, pool, B)
    st = streams_of(wl, pool)
    grad = grad_grid(11, B, 640)
    with P.EmbeddingShard(pool, B, weight_seed=seed) as sh:
        sh.load(st)
        sh.forward()
        g = torch.from_numpy(grad).cuda()
        sh.backward(g, LR, EPS)
        torch.cuda.synchronize()
        run_bwd_check(oracle, sh, pool, st, grad, seed, B)
        # rows never looked up are untouched
        t0 = pool[0]
        touched = set(np.unique(st[0][1]).tolist())
        probe = [r for r in range(0, t0.hash_size, max(1, t0.hash_size // 257)) if r not in touched][:64]
        assert np.array_equal(sh.read_rows(0, probe), weight_rows(seed, t0.id, probe, t0.dim))


@pytest.mark.parametrize("dims", [(4, 8, 12, 16, 20, 24, 32, 48), (64, 96, 128, 160, 192, 256), (384, 512, 1024)])
def test_mixed_dims_one_launch(P, oracle, cuda, dims):
    pool = P.generate_pool(1, len(dims), P.GeneratorConfig(hash_size_max=5e4, pooling_mean_target=30.0))
    for t, d in zip(pool, dims):
        t.dim = d
    B, seed = 300, 9
    wl = P.generate_workload(2, pool, B)
    st = streams_of(wl, pool)
    with P.EmbeddingShard(pool, B, weight_seed=seed) as sh:
        sh.load(st)
        sh.forward()
        pooled = sh.read_pooled()
        ref = oracle.forward_f64(to_oracle_tables(pool), B, st, wseed=seed)
        assert np.array_equal(pooled.astype(np.float64), ref)
        sh.backward(None, LR, EPS)
        run_bwd_check(oracle, sh, pool, st, pooled, seed, B)


def _handmade(B, lengths_per_table, rows_fn):
    streams = []
    for t, lens in enumerate(lengths_per_table):
        off = np.zeros(B + 1, dtype=np.int64)
        off[1:] = np.cumsum(lens)
        idx = rows_fn(t, int(off[-1]))
        streams.append((off, idx))
    return streams


@pytest.mark.parametrize("dim", [16, 128, 256])
def test_long_bags_hot_rows_empty_tables(P, oracle, cuda, dim):
    """Bags far longer than a chunk, a hot row spanning many chunks, runs of
    empty bags, bags exactly one chunk long, and a table with no lookups."""
    B = 64
    rng = np.random.default_rng(0)
    hash_sizes = [5000, 70, 10, 1000]
    # the device's chunk length for this batch (context.cu chunk_len_for): bags of
    # exactly one / two chunks and chunk-1 / chunk+1 exercise every carry case
    est = 4.0 * dim * (20000 + 4 * 2048 + 5000 + 50 * B)
    target = max(2048.0, min(262144.0, est / (148.0 * 24.0)))
    target = min(target, 262144.0 / (8 if dim == 16 else 1))  # 256 KB per warp unit of 32/GL chunks
    chunk = max(32, min(8192, int(target / (dim * 4.0)) // 32 * 32))
    lens = [
        np.array([0, 20000, 1, 0, 0, chunk, chunk, 2 * chunk + 1] + [3] * (B - 8)),
        np.array([chunk - 1, 1, chunk + 1] + [0] * (B - 4) + [5000]),
        np.zeros(B, dtype=np.int64),
        rng.integers(0, 50, size=B),
    ]

    def rows(t, n):
        if t == 1:
            return np.zeros(n, dtype=np.int64) + 3  # one hot row, every lookup
        r = rng.integers(0, hash_sizes[t], size=n)
        r[: n // 2] = 7  # hot row in the first half
        return r.astype(np.int64)

    st = _handmade(B, lens, rows)
    tables = [P.TableDesc(id=10 + t, dim=dim, hash_size=h, pooling_mean=1.0) for t, h in enumerate(hash_sizes)]
    seed = 4
    with P.EmbeddingShard(tables, B, weight_seed=seed) as sh:
        sh.load(st)
        sh.forward()
        pooled = sh.read_pooled()
        ref = oracle.forward_f64(to_oracle_tables(tables), B, st, wseed=seed)
        ok, worst = fp_close(pooled, ref, rtol=0, atol=0)
        assert ok, f"forward not bit-exact ({worst})"
        sh.backward(None, LR, EPS)
        run_bwd_check(oracle, sh, tables, st, pooled, seed, B)


def test_multistep_dense_against_oracle(P, oracle, cuda):
    """Three fwd/bwd steps with grad = pooled (loss 1/2|pooled|^2), weights
    evolving in place; oracle keeps dense fp32 tables updated from fp64 math."""
    pool = P.generate_pool(5, 5, P.GeneratorConfig(dim_choices=(8, 32, 64), hash_size_max=3000,
                                                  pooling_mean_target=25.0))
    B, seed = 200, 13
    wl = P.generate_workload(5, pool, B)
    st = streams_of(wl, pool)
    W = [weight_rows(seed, t.id, np.arange(t.hash_size), t.dim) for t in pool]
    M = [np.zeros(t.hash_size, dtype=np.float32) for t in pool]
    ot = to_oracle_tables(pool)
    with P.EmbeddingShard(pool, B, weight_seed=seed) as sh:
        sh.load(st)
        for step in range(3):
            sh.forward()
            pooled = sh.read_pooled()
            ref = oracle.forward_f64(ot, B, st, dense=W)
            # after step 0 the weights leave the exact grid: bound by the bag's sum of |terms|
            terms = oracle.forward_f64(ot, B, st, dense=[np.abs(w) for w in W])
            ok, worst = fp_close(pooled, ref, rtol=1e-5, atol=1e-7, scale=terms)
            assert ok, f"step {step}: forward off by {worst:.3g}x tolerance"
            sh.backward(None, LR, EPS)
            grad = ref.astype(np.float32)
            W_old = [w.copy() for w in W]
            for t in range(len(pool)):
                oracle.backward_adagrad_f64(ot[t], B, *st[t], grad, sh.cols[t], LR, EPS, W=W[t], M=M[t])
            for t, tab in enumerate(pool):
                allrows = np.arange(tab.hash_size)
                scale = np.maximum(np.abs(W_old[t]), np.abs(W_old[t] - W[t]))
                ok, worst = fp_close(sh.read_rows(t, allrows), W[t], rtol=1e-5, atol=1e-6, scale=scale)
                assert ok, f"step {step} table {tab.id}: weights off by {worst:.3g}x"


def test_step_loss(P, cuda):
    pool = P.generate_pool(0, 4, P.GeneratorConfig(hash_size_max=1e4))
    B = 1000
    wl = P.generate_workload(0, pool, B)
    with P.EmbeddingShard(pool, B, weight_seed=1) as sh:
        sh.load(wl)
        sh.forward()
        pooled = sh.read_pooled().astype(np.float64)
        loss = sh.step(LR, EPS, want_loss=True)
        assert abs(loss - 0.5 * (pooled ** 2).sum()) <= 1e-5 * max(1.0, loss)


def test_load_validation_errors(P, cuda):
    tables = [P.TableDesc(id=3, dim=16, hash_size=10), P.TableDesc(id=8, dim=16, hash_size=20)]
    B = 4
    good = [(np.array([0, 1, 2, 3, 4]), np.array([1, 2, 3, 4])), (np.array([0, 0, 1, 1, 2]), np.array([5, 19]))]
    with P.EmbeddingShard(tables, B) as sh:
        sh.load(good)
        with pytest.raises(P.OffsetError, match="table 8: offsets must start at 0, got 1"):
            sh.load([good[0], (np.array([1, 1, 1, 1, 2]), np.array([5, 19]))])
        with pytest.raises(P.OffsetError, match="table 3: offsets must be nondecreasing at entry 2"):
            sh.load([(np.array([0, 2, 1, 3, 4]), np.array([1, 2, 3, 4])), good[1]])
        with pytest.raises(P.OffsetError, match="table 8: final offset 2 != index count 3"):
            sh.load([good[0], (np.array([0, 0, 1, 1, 2]), np.array([5, 19, 1]))])
        with pytest.raises(P.IndexError_, match=r"table 8: index 20 out of range \[0, 20\)"):
            sh.load([good[0], (np.array([0, 0, 1, 1, 2]), np.array([5, 20]))])
        with pytest.raises(P.IndexError_, match=r"table 3: index -1 out of range"):
            sh.load([(np.array([0, 1, 2, 3, 4]), np.array([1, -1, 3, 4])), good[1]])
        with pytest.raises(P.StateError):
            sh.forward()  # failed load leaves no batch loaded
        sh.load(good)
        sh.forward()


def test_bad_dims_rejected(P, cuda):
    with pytest.raises(P.ConfigError):
        P.EmbeddingShard([P.TableDesc(id=0, dim=6, hash_size=10)], 4)
    with pytest.raises(P.ConfigError):
        P.EmbeddingShard([P.TableDesc(id=0, dim=2048, hash_size=10)], 4)


def test_measure_protocol_and_measure_plan(P, cuda):
    pool = P.generate_pool(0, 12, P.GeneratorConfig(hash_size_max=1e5))
    B = 4096
    wl = P.generate_workload(0, pool, B)
    with P.EmbeddingShard(pool, B) as sh:
        sh.load(wl)
        ms = sh.measure(2, 5, 1, True)
        assert ms > 0
        with pytest.raises(P.ConfigError, match="need measure - 2\\*trim >= 1"):
            sh.measure(1, 4, 2, True)
    task = P.ShardingTask(pool, 3, [sum(t.size_bytes() for t in pool)] * 3)
    plan = P.greedy_shard(task, P.HeuristicKind.kLookupGreedy)
    costs = P.measure_plan(plan, task, wl, P.BenchConfig(warmup=1, measure=3, trim=1))
    assert len(costs) == 3 and all(c > 0 for c in costs)
    # an empty shard reports its (small, positive) launch time, not 0
    empty = P.ShardingPlan([0] * len(pool))
    c2 = P.measure_plan(empty, task, wl, P.BenchConfig(warmup=1, measure=3, trim=1))
    assert c2[1] >= 0 and c2[0] > c2[1]
    other = P.generate_pool(1, 13)[12:]
    with pytest.raises(P.LookupError_):
        P.measure_plan(P.ShardingPlan([0]), P.ShardingTask(other, 1, [10 ** 12]), wl,
                       P.BenchConfig(warmup=0, measure=1, trim=0))
    with pytest.raises(P.ConfigError):
        P.measure_plan(P.ShardingPlan([5] * len(pool)), task, wl)


def test_cfg2_full_size_properties(P, cuda):
    """BASELINE cfg 2 at full size (50 tables, dim 128, B=65536): size-independent
    checks — column sums of the pooled output equal sum over unique rows of
    count * W[row] (exact on the weight grid, checked per table in fp64) and
    the momentum of sampled unique rows equals |g_r|^2/D."""
    pool = P.generate_pool(0, 856)[:50]
    for t in pool:
        t.dim = 128
    B, seed = 65536, 0
    wl = P.generate_workload(0, pool, B)
    with P.EmbeddingShard(pool, B, weight_seed=seed) as sh:
        sh.load(wl)
        sh.forward()
        pooled = sh.read_pooled()
        rng = np.random.default_rng(0)
        for t in rng.choice(len(pool), size=6, replace=False):
            tab = pool[t]
            idx = wl.find(tab.id).indices
            rows, counts = np.unique(idx, return_counts=True)
            W = weight_rows(seed, tab.id, rows, tab.dim).astype(np.float64)
            want = (W * counts[:, None]).sum(0)
            got = pooled[:, sh.cols[t]:sh.cols[t] + 128].astype(np.float64).sum(0)
            assert np.allclose(got, want, rtol=1e-9, atol=1e-6)
        sh.backward(None, LR, EPS)
        for t in rng.choice(len(pool), size=3, replace=False):
            tab = pool[t]
            s = wl.find(tab.id)
            bags = bag_ids(s.offsets)
            rows, inv = np.unique(s.indices, return_inverse=True)
            order = np.argsort(inv, kind="stable")
            bounds = np.searchsorted(inv[order], np.arange(len(rows) + 1))
            pick = rng.choice(len(rows), size=min(200, len(rows)), replace=False)
            G = pooled[:, sh.cols[t]:sh.cols[t] + 128].astype(np.float64)
            got = sh.read_momentum(int(t), rows[pick])
            for q, k in enumerate(pick):
                g = G[bags[order[bounds[k]:bounds[k + 1]]]].sum(0)
                want = (g @ g) / 128
                assert abs(got[q] - want) <= 1e-5 * want + 1e-30


def test_async_staging_pipeline_matches_sync_load(P, oracle, cuda):
    """as_stage_* / as_commit_staged double buffering gives the same results as
    the synchronous load, across alternating batches, and reports a bad batch."""
    pool = P.generate_pool(2, 5, P.GeneratorConfig(dim_choices=(16, 64), hash_size_max=2e4))
    B, seed = 256, 1
    wls = [P.generate_workload(s, pool, B) for s in (10, 11, 12)]
    ot = to_oracle_tables(pool)
    with P.EmbeddingShard(pool, B, weight_seed=seed) as sh:
        sh.stage(wls[0])
        sh.stage(wls[1])
        with pytest.raises(P.StateError):
            sh.stage(wls[2])  # two slots only
        for k in range(3):
            sh.commit()
            with pytest.raises(P.StateError):
                if k == 0:
                    sh.stage(wls[2])  # slot of the current batch is busy, the other is staged
                else:
                    sh.commit()  # nothing staged
            if k == 1:
                sh.stage(wls[2])
            sh.forward()
            got = sh.read_pooled()
            st = streams_of(wls[k], pool)
            assert np.array_equal(got.astype(np.float64), oracle.forward_f64(ot, B, st, wseed=seed))
        bad = [(wls[0].find(t.id).offsets, wls[0].find(t.id).indices.copy()) for t in pool]
        bad[3][1][0] = pool[3].hash_size
        sh.stage(bad)
        with pytest.raises(P.IndexError_, match=f"table {pool[3].id}: index {pool[3].hash_size} out of range"):
            sh.commit()
        with pytest.raises(P.StateError):
            sh.forward()


def _features_np(tab, idx, B):
    """extract_features raw layout (tables.hpp:344-386), restated with numpy."""
    f = np.zeros(21)
    f[0], f[1], f[2] = tab.dim, tab.hash_size, len(idx) / B
    f[3] = tab.dim * tab.hash_size * tab.bytes_per_param / 1024.0 ** 3
    if len(idx):
        _, counts = np.unique(idx, return_counts=True)
        bins = np.zeros(17)
        for c in counts:
            b = 0 if c <= 1 else min(int(c - 1).bit_length(), 16)
            bins[b] += 1
        f[4:] = bins / len(counts)
    return f


def test_gpu_cost_model_features(P, cuda):
    """the 21 raw features of extract_features from the GPU sort,
    exact (integer bins, same division) — including a hot row > 32768 hits."""
    pool = P.generate_pool(0, 12, P.GeneratorConfig(hash_size_max=3e5, pooling_mean_target=30.0))
    B = 4096
    wl = P.generate_workload(0, pool, B)
    st = streams_of(wl, pool)
    extra = P.TableDesc(id=99, dim=16, hash_size=50, pooling_mean=20.0)
    off = np.arange(B + 1, dtype=np.int64) * 20
    idx = np.zeros(B * 20, dtype=np.int64)
    idx[::7] = 3
    tables, streams = pool + [extra], st + [(off, idx)]
    with P.EmbeddingShard(tables, B) as sh:
        sh.load(streams)
        got = sh.features()
        want = np.stack([_features_np(t, s[1], B) for t, s in zip(tables, streams)])
        assert np.array_equal(got, want)
        sh.forward()  # with the side-stream sort in flight
        assert np.array_equal(sh.features(), want)


@pytest.mark.parametrize("world,extra", [(2, 0), (4, 3), (3, 1)])
def test_fused_exchange_peer_stores(world, extra):
    """Fused forward exchange (as_set_peer_outputs_v), G virtual ranks on one GPU:
    every owner's forward writes its pooled rows straight into the sample
    owners' receive buffers; each receive buffer must equal what the NCCL
    all-to-all of the plain [B, SD_k] outputs delivers (bit-exact), including
    the zero rows of empty bags — also for uneven sample splits (B % G != 0)."""
    import torch

    import paper_2208_06399_b200 as P
    from paper_2208_06399_b200.sharded import a2a_layout, peer_bases

    pool = P.generate_pool(3, 12, P.GeneratorConfig(dim_choices=(8, 16, 64, 132), hash_size_max=3e4,
                                                   pooling_mean_target=6.0))
    B = 64 * world + extra
    wl = P.generate_workload(5, pool, B)
    task = P.ShardingTask(pool, world, [1 << 40] * world)
    plan = P.random_shard(task, 1)
    lay = a2a_layout(task, plan, B)
    members = plan.shard_member_indices(task)
    recv = [torch.full((lay.rows(q) * sum(lay.shard_dims),), float("nan"), device="cuda") for q in range(world)]
    plain = []
    shards = []
    for k in range(world):
        tabs = [pool[i] for i in members[k]]
        sh = P.EmbeddingShard(tabs, B, device=0, weight_seed=11)
        sh.load(streams_of(wl, tabs))
        sh.forward()
        torch.cuda.synchronize()
        plain.append(sh.read_pooled())
        sh.set_peer_outputs(peer_bases(lay, k, [r.data_ptr() for r in recv]), lay.row_start)
        shards.append(sh)
    for sh in shards:
        sh.forward()
    torch.cuda.synchronize()
    for q in range(world):
        got = recv[q].cpu().numpy()
        r0, r1 = lay.row_start[q], lay.row_start[q + 1]
        for k in range(world):
            o = lay.recv_offset(k, q)
            blk = got[o:o + lay.rows(q) * lay.shard_dims[k]].reshape(lay.rows(q), lay.shard_dims[k])
            assert np.array_equal(blk, plain[k][r0:r1]), (q, k)
    # the fused forward refuses an implicit gradient and the single-call step
    with pytest.raises(P.StateError):
        shards[0].backward(None)
    for sh in shards:
        sh.set_peer_outputs([], 0)
        sh.close()


@pytest.mark.parametrize("dims", [(4, 16, 32, 64), (128, 132, 256, 512)])
def test_fp16_weight_storage(P, oracle, cuda, dims):
    """AS_WEIGHTS_FP16 (bytes_per_param 2). Forward: bit-exact
    (the grid init k*2^-12, |k| <= 512, is exact in fp16 and accumulation is
    fp32). Backward: the fp32 update rounded to nearest fp16, so the updated
    rows match the fp64 oracle within half an fp16 ulp (2^-11 relative) plus
    the fp32 bound; momentum stays fp32 (1e-5)."""
    pool = P.generate_pool(4, len(dims), P.GeneratorConfig(hash_size_max=4e4, pooling_mean_target=25.0))
    for t, d in zip(pool, dims):
        t.dim = d
    B, seed = 256, 6
    wl = P.generate_workload(3, pool, B)
    st = streams_of(wl, pool)
    with P.EmbeddingShard(pool, B, weight_seed=seed, weights="fp16") as sh:
        assert sh.info().weight_bytes == 2
        sh.load(st)
        sh.forward()
        pooled = sh.read_pooled()
        ref = oracle.forward_f64(to_oracle_tables(pool), B, st, wseed=seed)
        assert np.array_equal(pooled.astype(np.float64), ref)
        sh.backward(None, LR, EPS)
        for t, tab in enumerate(pool):
            r = oracle.backward_adagrad_f64(to_oracle_tables([tab])[0], B, *st[t], pooled, sh.cols[t], LR, EPS,
                                            wseed=seed)
            if len(r["rows"]) == 0:
                continue
            w = sh.read_rows(t, r["rows"]).astype(np.float64)
            w_old = weight_rows(seed, tab.id, r["rows"], tab.dim).astype(np.float64)
            scale = np.maximum(np.abs(w_old), np.abs(w_old - r["w"]))
            tol = 2.0 ** -11 * np.abs(r["w"]) * 1.001 + 1e-5 * scale + 2.0 ** -24
            err = np.abs(w - r["w"])
            assert (err <= tol).all(), f"table {tab.id}: fp16 rows off by {float((err / tol).max()):.3g}x tolerance"
            assert np.array_equal(w, w.astype(np.float16).astype(np.float64))  # stored values are fp16
            ok, worst = fp_close(sh.read_momentum(t, r["rows"]), r["m"])
            assert ok, f"table {tab.id}: momentum off by {worst:.3g}x tolerance"


def test_gpu_side_narrowing_and_validation(P, oracle, cuda, monkeypatch):
    """ASB_RAW_EIGHTHS=8: every index piece of a pinned batch goes host->device
    as int64 and is narrowed + validated on the GPU (narrow_validate_kernel).
    Same device rows, bit-exact forward, and the same first error (table,
    check, entry order; load_workload's message) as the host path."""
    monkeypatch.setenv("ASB_RAW_EIGHTHS", "8")
    pool = P.generate_pool(6, 5, P.GeneratorConfig(dim_choices=(16, 64), hash_size_max=3e4))
    B, seed = 256, 2
    wl = P.generate_workload(4, pool, B).pin()
    st = streams_of(wl, pool)
    with P.EmbeddingShard(pool, B, weight_seed=seed) as sh:
        sh.load(wl)
        sh.forward()
        assert np.array_equal(sh.read_pooled().astype(np.float64),
                              oracle.forward_f64(to_oracle_tables(pool), B, st, wseed=seed))
        row0 = np.cumsum([0] + [t.hash_size for t in pool])[:-1]
        glob = np.concatenate([idx + r0 for (_, idx), r0 in zip(st, row0)])
        assert np.array_equal(sh.read_buffer(P.device.GLOBAL_ROWS), glob)
        t3, t4 = pool[3], pool[4]
        idx3, idx4 = wl.find(t3.id).indices, wl.find(t4.id).indices
        keep = (idx3[2], idx3[5], idx4[1])
        idx3[5], idx3[2], idx4[1] = t3.hash_size + 7, -3, t4.hash_size
        sh.stage(wl)
        with pytest.raises(P.IndexError_, match=rf"table {t3.id}: index -3 out of range \[0, {t3.hash_size}\)"):
            sh.commit()
        idx3[2] = keep[0]
        sh.stage(wl)
        with pytest.raises(P.IndexError_, match=rf"table {t3.id}: index {t3.hash_size + 7} out of range"):
            sh.commit()
        idx3[5], idx4[1] = keep[1], keep[2]
        sh.load(wl)
        sh.forward()
        assert np.array_equal(sh.read_pooled().astype(np.float64),
                              oracle.forward_f64(to_oracle_tables(pool), B, st, wseed=seed))


def test_cfg4_shard_full_size_properties(P, cuda):
    """An 8-GPU-sized slice of BASELINE cfg 4 at full batch (every 8th table of
    pool856: 107 tables, dims 16/32, B = 65,536): narrow lane layouts, the
    table-segmented sort (1-3 passes per table), in-warp and fixup completion
    of hot rows. Bit-exact: each sampled table's sorted (row, bag) order equals
    numpy's stable argsort; the pooled column sums equal sum(count * W[row]);
    the momentum of sampled rows equals |g_r|^2 / D."""
    pool = P.generate_pool(0, 856)[::8]
    B, seed = 65536, 0
    wl = P.generate_workload(0, pool, B)
    with P.EmbeddingShard(pool, B, weight_seed=seed) as sh:
        sh.load(wl)
        sh.forward()
        pooled = sh.read_pooled()
        sh.backward(None, LR, EPS)
        srows = sh.read_buffer(P.device.SORTED_ROWS)
        sbags = sh.read_buffer(P.device.SORTED_BAGS)
        row0 = np.cumsum([0] + [t.hash_size for t in pool])[:-1]
        start = np.cumsum([0] + [len(wl.find(t.id).indices) for t in pool])
        rng = np.random.default_rng(1)
        for t in rng.choice(len(pool), size=8, replace=False):
            tab = pool[t]
            s = wl.find(tab.id)
            bags = bag_ids(s.offsets)
            order = np.argsort(s.indices, kind="stable")
            a, b = start[t], start[t + 1]
            assert np.array_equal(srows[a:b], s.indices[order] + row0[t]), tab.id
            assert np.array_equal(sbags[a:b], bags[order]), tab.id
            rows, counts = np.unique(s.indices, return_counts=True)
            W = weight_rows(seed, tab.id, rows, tab.dim).astype(np.float64)
            got = pooled[:, sh.cols[t]:sh.cols[t] + tab.dim].astype(np.float64).sum(0)
            assert np.allclose(got, (W * counts[:, None]).sum(0), rtol=1e-9, atol=1e-6), tab.id
            inv = np.searchsorted(rows, s.indices[order])
            bounds = np.searchsorted(inv, np.arange(len(rows) + 1))
            pick = np.concatenate([np.argsort(-counts)[:5], rng.choice(len(rows), size=min(100, len(rows)), replace=False)])
            G = pooled[:, sh.cols[t]:sh.cols[t] + tab.dim].astype(np.float64)
            mom = sh.read_momentum(int(t), rows[pick])
            for q, k in enumerate(pick):
                g = G[bags[order[bounds[k]:bounds[k + 1]]]].sum(0)
                want = (g @ g) / tab.dim
                assert abs(mom[q] - want) <= 1e-5 * want + 1e-30, (tab.id, rows[k], counts[k])


def test_backward_without_forward_after_load(P, oracle, cuda):
    """as_backward_rowwise_adagrad straight after a load (no as_forward of this
    batch): the sort's bag ids must come from THIS batch (K4 runs in ids-only
    mode), not from the previous batch's forward."""
    torch = cuda
    pool = P.generate_pool(2, 6, P.GeneratorConfig(dim_choices=(16, 64), hash_size_max=2e4))
    B, seed = 700, 21
    wl_a = P.generate_workload(1, pool, B)
    wl_b = P.generate_workload(2, pool, B)
    st_b = streams_of(wl_b, pool)
    grad = grad_grid(5, B, sum(t.dim for t in pool))
    with P.EmbeddingShard(pool, B, weight_seed=seed) as sh:
        sh.load(wl_a)
        sh.forward()  # bag ids of batch A in the device buffers
        sh.load(st_b)
        sh.backward(torch.from_numpy(grad).cuda(), LR, EPS)
        torch.cuda.synchronize()
        run_bwd_check(oracle, sh, pool, st_b, grad, seed, B)


def test_sort_one_to_four_digit_passes(P, oracle, cuda):
    """K2 over tables needing 1, 2, 3 and 4 digit passes (hash 200 / 3e4 / 3e6 /
    2e7 rows), tables spanning many superblocks (>= 65,536 lookups each), bags
    of one lookup (thousands of bags per sort tile: the bag-id marking takes
    several rounds), long runs of empty bags and a Zipf-hot row: sorted
    (row, bag) order bit-exact against numpy's stable argsort, then the
    backward within tolerance."""
    torch = cuda
    B = 20000
    rng = np.random.default_rng(7)
    hash_sizes = [200, 30000, 3_000_000, 20_000_000, 5000]
    lens = [
        rng.integers(0, 8, size=B),                          # short bags, 1 pass
        np.where(rng.random(B) < 0.6, 0, rng.integers(1, 40, size=B)),  # 60 % empty bags
        np.ones(B, dtype=np.int64),                          # one lookup per bag
        rng.integers(0, 12, size=B),
        np.concatenate([np.zeros(B // 2, dtype=np.int64), rng.integers(0, 30, size=B - B // 2)]),
    ]

    def rows(t, n):
        r = rng.zipf(1.3, size=n) % hash_sizes[t]
        r[::5] = rng.integers(0, hash_sizes[t], size=len(r[::5]))
        return r.astype(np.int64)

    st = _handmade(B, lens, rows)
    tables = [P.TableDesc(id=40 + t, dim=d, hash_size=h, pooling_mean=1.0)
              for t, (h, d) in enumerate(zip(hash_sizes, (16, 32, 64, 128, 8)))]
    seed = 13
    grad = grad_grid(3, B, sum(t.dim for t in tables))
    with P.EmbeddingShard(tables, B, weight_seed=seed) as sh:
        sh.load(st)
        sh.backward(torch.from_numpy(grad).cuda(), LR, EPS)
        torch.cuda.synchronize()
        row_off = np.cumsum([0] + hash_sizes)[:-1]
        glob = np.concatenate([i + r0 for (_, i), r0 in zip(st, row_off)]).astype(np.int64)
        bags = np.concatenate([bag_ids(o) for o, _ in st])
        order = np.argsort(glob, kind="stable")
        assert np.array_equal(sh.read_buffer(P.device.SORTED_ROWS).astype(np.int64), glob[order])
        assert np.array_equal(sh.read_buffer(P.device.SORTED_BAGS), bags[order])
        run_bwd_check(oracle, sh, tables, st, grad, seed, B)


def test_subset_shard_on_parent_storage(P, oracle, cuda):
    """as_create_subset: a shard over some of a parent's tables, on the parent's
    weight and momentum storage. A step through it equals a standalone shard of
    the same tables (same seed -> same initial rows) bit for bit, writes the
    update into the PARENT's rows, and leaves the other tables untouched; the
    measured-cost hook (ShardCostService) times shards this way."""
    pool = P.generate_pool(4, 6, P.GeneratorConfig(dim_choices=(16, 32, 64, 128), hash_size_max=3e4))
    B, seed = 600, 17
    wl = P.generate_workload(3, pool, B)
    pos = [4, 1, 2]
    sub_tables = [pool[p] for p in pos]
    with P.EmbeddingShard(pool, B, weight_seed=seed) as parent, P.EmbeddingShard(sub_tables, B, weight_seed=seed) as ref:
        sub = parent.subset(pos)
        try:
            assert sub.sum_dim == sum(t.dim for t in sub_tables)
            sub.load(wl)
            ref.load(wl)
            l_sub = sub.step(LR, EPS, want_loss=True)
            l_ref = ref.step(LR, EPS, want_loss=True)
            assert l_sub == pytest.approx(l_ref, rel=1e-9)  # per-warp partials added in any order
            assert np.array_equal(sub.read_pooled(), ref.read_pooled())
            for i, p in enumerate(pos):
                rows = np.arange(pool[p].hash_size)
                assert np.array_equal(parent.read_rows(p, rows), ref.read_rows(i, rows)), pool[p].id
                assert np.array_equal(parent.read_momentum(p, rows), ref.read_momentum(i, rows)), pool[p].id
            for p in (0, 3, 5):  # not in the subset: still the initial rows
                rows = np.arange(0, pool[p].hash_size, 97)
                assert np.array_equal(parent.read_rows(p, rows), weight_rows(seed, pool[p].id, rows, pool[p].dim))
            assert sub.measure(1, 3, 1) > 0.0
            # another subset through the same context (grow-only buffers)
            sub.retarget([0, 3, 5, 2])
            sub.load(wl)
            ref2_tables = [pool[p] for p in (0, 3, 5, 2)]
            with P.EmbeddingShard(ref2_tables, B, weight_seed=seed) as ref2:
                ref2.load(wl)
                sub.forward()
                ref2.forward()
                got, want = sub.read_pooled(), ref2.read_pooled()
                # table 2 was updated by the first step in the parent: compare the untouched ones
                for i, p in enumerate((0, 3, 5)):
                    c = sub.cols[i]
                    assert np.array_equal(got[:, c:c + pool[p].dim], want[:, c:c + pool[p].dim]), pool[p].id
        finally:
            sub.close()
        with pytest.raises(P.ConfigError):
            parent.subset([1, 1])
        with pytest.raises(P.ConfigError):
            parent.subset([6])
