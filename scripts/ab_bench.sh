#!/bin/bash
# bench.py headline (graph replay) + stream-launched value for library variants in build/
mkdir -p gpurun_out
for v in $1; do
  echo "=== bench $v"
  SS_B200_LIB=$PWD/build/$v.so python bench.py --steps 100 --warmup 10 2>gpurun_out/abb_$v.err | tee gpurun_out/abb_$v.json | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'stream', round(d['stream_launches']['value'],1), 'e2e', round(d['e2e']['value'],1), 'plugin', round(d['e2e_plugin']['value'],1), 'k_raster', round(d['roofline']['avg_launch_ms']*1000,1), 'launches', d['gpu_launches'])"
done
