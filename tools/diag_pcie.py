"""Host->device bandwidth of one e2e batch under the loads the pipeline puts
beside it: alone, beside a memory-bound kernel loop, beside the host narrowing
(as_stage_workload on the other slot), and the int64 streams copied raw."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_06399_b200 as P  # noqa: E402


def h2d(src, dst, stream, reps=5):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        ev0.record(stream)
        with torch.cuda.stream(stream):
            dst.copy_(src, non_blocking=True)
        ev1.record(stream)
        ev1.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    n32 = 36_484_624  # cfg2 lookups (int32 rows)
    host32 = torch.empty(n32, dtype=torch.int32).pin_memory()
    host64 = torch.empty(n32, dtype=torch.int64).pin_memory()
    host32.fill_(1)
    host64.fill_(1)
    dev32 = torch.empty(n32, dtype=torch.int32, device="cuda")
    dev64 = torch.empty(n32, dtype=torch.int64, device="cuda")
    cs = torch.cuda.Stream()
    out = {}
    ms = h2d(host32, dev32, cs)
    out["int32_alone"] = (ms, host32.numel() * 4 / ms / 1e6)
    ms = h2d(host64, dev64, cs)
    out["int64_alone"] = (ms, host64.numel() * 8 / ms / 1e6)

    # beside a memory-bound device loop (D2D copies of 2 GB on another stream)
    a = torch.empty(1 << 29, dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    ks = torch.cuda.Stream()
    stop = threading.Event()

    def loop():
        with torch.cuda.stream(ks):
            while not stop.is_set():
                for _ in range(8):
                    b.copy_(a)
                ks.synchronize()

    th = threading.Thread(target=loop)
    th.start()
    time.sleep(0.2)
    ms = h2d(host32, dev32, cs)
    out["int32_beside_d2d_loop"] = (ms, host32.numel() * 4 / ms / 1e6)
    stop.set()
    th.join()
    del a, b

    # beside the embedding step itself (device-resident batch, back to back)
    tables, B, _ = bench.build_workload(P, "cfg2")
    wl = P.generate_workload(0, tables, B).pin()
    sh = P.EmbeddingShard(tables, B)
    s = torch.cuda.current_stream()
    sh.load(wl)
    stop = threading.Event()

    def steps():
        while not stop.is_set():
            sh.step(0.01, 1e-8, want_loss=False, stream=s)
            s.synchronize()

    th = threading.Thread(target=steps)
    th.start()
    time.sleep(0.2)
    ms = h2d(host32, dev32, cs)
    out["int32_beside_emb_steps"] = (ms, host32.numel() * 4 / ms / 1e6)
    stop.set()
    th.join()

    # host narrowing alone (stage + commit, no kernels)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        sh.stage(wl)
        sh.commit(s)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    ts.sort()
    out["stage_commit_alone_ms"] = ts[2]
    # H2D beside host narrowing of the other slot
    stop = threading.Event()

    def staging():
        while not stop.is_set():
            sh.stage(wl)
            sh.commit(s)
            torch.cuda.synchronize()

    th = threading.Thread(target=staging)
    th.start()
    time.sleep(0.2)
    ms = h2d(host32, dev32, cs)
    out["int32_beside_staging"] = (ms, host32.numel() * 4 / ms / 1e6)
    stop.set()
    th.join()
    for k, v in out.items():
        if isinstance(v, tuple):
            print(f"{k:28s} {v[0]:7.2f} ms  {v[1]:6.1f} GB/s")
        else:
            print(f"{k:28s} {v:7.2f} ms")


if __name__ == "__main__":
    main()
