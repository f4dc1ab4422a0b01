"""Where does the e2e pipeline lose its overlap? Commit wait (= staging not done
yet) after staging ran beside: nothing (sleep), a torch D2D loop, our step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_06399_b200 as P  # noqa: E402


def main():
    tables, B, _ = bench.build_workload(P, "cfg2")
    wl = P.generate_workload(0, tables, B).pin()
    sh = P.EmbeddingShard(tables, B)
    s = torch.cuda.current_stream()
    sh.stage(wl)
    sh.commit(s)
    a = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)

    def run(label, beside, reps=5):
        res = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sh.stage(wl)
            t1 = time.perf_counter()
            beside()
            t2 = time.perf_counter()
            sh.commit(s)
            t3 = time.perf_counter()
            torch.cuda.synchronize()
            t4 = time.perf_counter()
            res.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t0)))
        res.sort(key=lambda r: r[3])
        r = res[len(res) // 2]
        print(f"{label:22s} stage-call {r[0]:5.2f}  beside {r[1]:5.2f}  commit-wait {r[2]:5.2f}  total {r[3]:5.2f} ms",
              flush=True)

    run("nothing", lambda: None)
    run("sleep 4ms", lambda: time.sleep(0.004))

    def d2d():
        for _ in range(3):
            b.copy_(a)
        s.synchronize()

    run("torch d2d ~4ms", d2d)
    run("emb step", lambda: sh.step(0.01, 1e-8, want_loss=True, stream=s))

    def spin():
        t = time.perf_counter()
        while time.perf_counter() - t < 0.004:
            pass

    run("host spin 4ms", spin)


if __name__ == "__main__":
    main()
