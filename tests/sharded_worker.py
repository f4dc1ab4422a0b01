"""One rank of the multi-process sharded-step parity test (test_sharded_multiproc.py).

Runs the C-ABI sharded step (as_comm: fused peer-store forward exchange, device
barrier, gradient push or NCCL, K2/K3) on this rank's shard and checks, against
the fp64 oracle of ALL tables on one process: this rank's receive buffer
(bit-exact), the loss, and every updated row + momentum of its own tables.
torch.distributed (gloo) is only the control plane (unique id / handle blobs).
Prints one JSON line."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import torch.distributed as dist

    import paper_2208_06399_b200 as P
    from helpers import fp_close, to_oracle_tables, weight_rows
    from oracle import Oracle
    from paper_2208_06399_b200.sharded import a2a_layout, connect, local_batch, local_tables, recv_table_rows

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    mode, use_nccl = int(os.environ["ASB_MODE"]), os.environ.get("ASB_NCCL") == "1"
    dev = rank if os.environ.get("ASB_ONE_GPU") != "1" else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    LR, EPS, SEED = 0.01, 1e-8, 3
    pool = P.generate_pool(4, 11, P.GeneratorConfig(dim_choices=(16, 32, 64, 128), hash_size_max=4e4,
                                                   pooling_mean_target=12.0))
    B = 64 * world + 3  # uneven sample split
    task = P.ShardingTask(pool, world, [1 << 40] * world)
    plan = P.random_shard(task, 5)
    lay = a2a_layout(task, plan, B)
    mine = local_tables(task, plan, rank)
    wl = P.generate_workload(0, mine, B)
    out = {"rank": rank, "ok": True, "errors": []}
    with P.EmbeddingShard(mine, B, device=dev, weight_seed=SEED) as sh:
        sh.load(wl)
        comm = connect(sh, lay, rank, world, mode=mode, use_nccl=use_nccl,
                       host_barrier=os.environ.get("ASB_ONE_GPU") == "1")
        loss = comm.step(LR, EPS, want_loss=True)
        torch.cuda.synchronize()
        recv = comm.recv_tensor().cpu().numpy()
        o = Oracle()
        wl_all = P.generate_workload(0, pool, B)
        st_all = [(wl_all.find(t.id).offsets, wl_all.find(t.id).indices) for t in pool]
        full = o.forward_f64(to_oracle_tables(pool), B, st_all, wseed=SEED)
        cols = np.cumsum([0] + [t.dim for t in pool])
        r0, r1 = lay.row_start[rank], lay.row_start[rank + 1]
        for i, t in enumerate(pool):
            got = recv_table_rows(lay, recv, rank, i)
            if not np.array_equal(got.astype(np.float64), full[r0:r1, cols[i]:cols[i] + t.dim]):
                out["ok"] = False
                out["errors"].append(f"recv rows of table {t.id}")
        want_loss = 0.5 * float((recv.astype(np.float64) ** 2).sum())
        if abs(loss - want_loss) > 1e-9 * max(1.0, want_loss):
            out["ok"] = False
            out["errors"].append(f"loss {loss} != {want_loss}")
        members = plan.shard_member_indices(task)[rank]
        for k, i in enumerate(members):
            t = pool[i]
            grad = full[:, cols[i]:cols[i] + t.dim].astype(np.float32)
            r = o.backward_adagrad_f64(to_oracle_tables([t])[0], B, *st_all[i], grad, 0, LR, EPS, wseed=SEED)
            if len(r["rows"]) == 0:
                continue
            w = sh.read_rows(k, r["rows"])
            w_old = weight_rows(SEED, t.id, r["rows"], t.dim).astype(np.float64)
            ok, worst = fp_close(w, r["w"], scale=np.maximum(np.abs(w_old), np.abs(w_old - r["w"])))
            okm, worstm = fp_close(sh.read_momentum(k, r["rows"]), r["m"])
            if not (ok and okm):
                out["ok"] = False
                out["errors"].append(f"table {t.id}: rows {worst:.3g}x, momentum {worstm:.3g}x tolerance")
        # more steps: barrier epochs, buffer reuse across steps
        for _ in range(5):
            comm.step(LR, EPS, want_loss=False)
        if use_nccl:
            # KJT all-to-all: every rank holds its samples of ALL tables; after the
            # exchange its shard must hold exactly its tables' whole-batch streams
            rows_before = sh.read_buffer(P.device.GLOBAL_ROWS)
            local = local_batch(st_all, lay.row_start, rank)
            comm.load_exchanged(pool, plan.assignment, local)
            sh.forward()
            torch.cuda.synchronize()
            if not np.array_equal(sh.read_buffer(P.device.GLOBAL_ROWS), rows_before):
                out["ok"] = False
                out["errors"].append("KJT exchange: device rows differ from the direct load")
            want_bags = np.concatenate([np.repeat(np.arange(B, dtype=np.int32), np.diff(st_all[i][0]))
                                        for i in plan.shard_member_indices(task)[rank]] or [np.zeros(0, np.int32)])
            if not np.array_equal(sh.read_buffer(P.device.BAG_IDS), want_bags):
                out["ok"] = False
                out["errors"].append("KJT exchange: bag segmentation differs")
        comm.step(LR, EPS, want_loss=True)
        i = comm.info()
        out["bytes_sent_fwd"], out["bytes_sent_bwd"] = int(i.bytes_sent_fwd), int(i.bytes_sent_bwd)
        out["has_nccl"] = int(i.has_nccl)
        comm.close()
    dist.barrier()
    dist.destroy_process_group()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
