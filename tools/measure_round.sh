#!/bin/bash
# One measurement pass on a GPU box (run under gpurun), tagged $1 (e.g. r2n):
# ncu launch lists and `ncu --set full` summaries of ONE step's kernels FIRST,
# so profiles/ncu_traffic.json carries the DRAM bytes of these very sources
# when the bench lines are taken (bench.py reports them as roofline.traffic
# only when the sources sha matches); then the bench lines, the GPU tests and
# smoke(). compute-sanitizer runs in calls of its own (tools/sanitize.sh, one
# tool per call).
# The .ncu-rep files stay on the box unless KEEP_REP=1 (gpurun copies back <= 64 MiB).
tag=${1:-run}
set -x
mkdir -p gpurun_out
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
# kernels per step: K4 + 3 sort kernels per digit pass (3 passes: tables up to 2^24 rows) + K1 + 3 fixups + K3 + 3 fixups
N=18
for w in cfg2 cfg4; do
  # each command under ncu has just exited 0 without it (B200_PROFILING.md)
  timeout 300 python bench.py --workload $w --steps 2 --warmup 3 --profile-only > gpurun_out/${tag}_plain_$w.log 2>&1 &&
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_$w.csv \
    python bench.py --workload $w --steps 2 --warmup 3 --profile-only > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/${tag}_launches_$w.csv gpurun_out/${tag}_launches_$w.txt \
    "ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --workload $w --steps 2 --warmup 3 --profile-only" > /dev/null
  rm -f gpurun_out/${tag}_launches_$w.csv
  # one whole step (the 4th, after 3 warm-up steps)
  timeout 300 python bench.py --workload $w --steps 1 --warmup 3 --profile-only > gpurun_out/${tag}_plain1_$w.log 2>&1 &&
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"seg_|sort_|bag_expand" -s $((3 * N)) -c $N \
    -o /tmp/prof_${tag}_$w python bench.py --workload $w --steps 1 --warmup 3 --profile-only > gpurun_out/${tag}_ncu_$w.log 2>&1
  python tools/ncu_summary.py /tmp/prof_${tag}_$w.ncu-rep gpurun_out/${tag}_ncu_full_$w.txt $w > /dev/null 2>&1
  [ "$KEEP_REP" = 1 ] && cp /tmp/prof_${tag}_$w.ncu-rep gpurun_out/
done
# the bench lines read the traffic of this capture
cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json
timeout 300 python bench.py > gpurun_out/${tag}_bench_cfg2.json 2> gpurun_out/${tag}_bench_cfg2.err
timeout 300 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2>&1
timeout 300 python bench.py --workload cfg4 --no-cpu > gpurun_out/${tag}_bench_cfg4.json 2> gpurun_out/${tag}_bench_cfg4.err
timeout 300 python bench.py --workload cfg3 --no-cpu --no-e2e > gpurun_out/${tag}_bench_cfg3.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.log 2>&1
ls -la gpurun_out
