#!/bin/bash
# A/B an environment knob: tools/ab_env.sh <workload> "NAME=VAL" ...
w=$1; shift
for e in "" "$@"; do
  env $e timeout 300 python bench.py --workload $w --no-cpu --no-e2e --steps 20 > gpurun_out/abe.json 2>gpurun_out/abe.err || tail -3 gpurun_out/abe.err
  python -c "
import json; d=json.load(open('gpurun_out/abe.json')); p=d['phase_ms_per_step']
print('%-14s %-6s step %.3f  k4 %.3f fwd %.3f bwd %.3f sort %.3f fixf %.3f fixb %.3f' % ('${e:-default}','$w',d['ms_per_step'],p['bag_expand'],p['fwd_segreduce'],p['bwd_segreduce_adagrad'],p['radix_sort'],p['fwd_fixup'],p['bwd_fixup']))"
done
