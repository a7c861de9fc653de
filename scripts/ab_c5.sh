#!/bin/bash
# C5 (10 M spheres, 1920x1080, d = 16, n_track = 32, tau = 0.01) per-kernel times for library variants in build/
mkdir -p gpurun_out
for v in $1; do
  echo "=== C5 $v"
  SS_B200_LIB=$PWD/build/$v.so python scripts/run_config.py --count 10000000 --width 1920 --height 1080 --d 16 --k 32 --tau 0.01 ${2:+--oracle-sample} 2>&1 | tee gpurun_out/abc5_$v.txt | tail -14
done
