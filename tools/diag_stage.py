import sys, time; sys.path.insert(0, '.')
import torch, numpy as np
import paper_2208_06399_b200 as P
import bench
tables, B, _ = bench.build_workload(P, "cfg2")
wl = P.generate_workload(0, tables, B).pin()
sh = P.EmbeddingShard(tables, B)
for i in range(3):
    t0 = time.perf_counter(); sh.stage(wl); t1 = time.perf_counter(); sh.commit(); t2 = time.perf_counter(); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"stage {1e3*(t1-t0):.2f} ms  commit(join) {1e3*(t2-t1):.2f} ms  sync {1e3*(t3-t2):.2f} ms")
import os; print('cpus', os.cpu_count())
