"""Where the end-to-end step's time goes (cfg2, one B200): host timestamps of
the pipelined loop bench.py's e2e runs (step / commit / stage per batch), then
the staging path alone (narrow + validate + H2D + commit) and the device step
alone. Used to tell a host-staging-bound e2e from a slow step.

  python tools/diag_e2e.py
"""
import sys, time, os
sys.path.insert(0, '.')
import torch
import paper_2208_06399_b200 as P
import bench
tables, B, _ = bench.build_workload(P, "cfg2")
wl = P.generate_workload(0, tables, B).pin()
sh = P.EmbeddingShard(tables, B)
s = torch.cuda.current_stream()
sh.stage(wl); sh.commit(s); sh.stage(wl)
for i in range(6):
    t0 = time.perf_counter(); loss = sh.step(0.01, 1e-8, want_loss=True, stream=s)
    t1 = time.perf_counter(); sh.commit(s)
    t2 = time.perf_counter(); sh.stage(wl)
    t3 = time.perf_counter()
    print(f"step {1e3*(t1-t0):6.2f}  commit {1e3*(t2-t1):6.2f}  stage {1e3*(t3-t2):5.2f}  total {1e3*(t3-t0):6.2f} ms")
sh.commit(s); torch.cuda.synchronize()
# copy alone (no compute): stage+commit+sync
for i in range(3):
    t0 = time.perf_counter(); sh.stage(wl); sh.commit(s); torch.cuda.synchronize(); print(f"stage+commit+sync alone {1e3*(time.perf_counter()-t0):.2f} ms")
# step alone
for i in range(3):
    t0 = time.perf_counter(); sh.step(0.01, 1e-8, want_loss=True, stream=s); print(f"step alone {1e3*(time.perf_counter()-t0):.2f} ms")
