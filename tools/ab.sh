#!/bin/bash
# A/B the tuning variants under paper_2208_06399_b200/variants on a GPU box.
# usage: tools/ab.sh <workload> [variant ...]   (run under gpurun)
w=$1; shift
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=paper_2208_06399_b200/variants/lib_$v.so; fi
  AUTOSHARD_B200_LIB=$lib timeout 300 python bench.py --workload $w --no-cpu --no-e2e --steps 20 > gpurun_out/ab_${w}_$v.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/ab_${w}_$v.json')); p=d['phase_ms_per_step']
print('%-8s %-6s step %.3f  fwd %.3f bwd %.3f sort %.3f fixf %.3f fixb %.3f' % ('$v','$w',d['ms_per_step'],p['fwd_segreduce'],p['bwd_segreduce_adagrad'],p['radix_sort'],p['fwd_fixup'],p['bwd_fixup']))"
done
