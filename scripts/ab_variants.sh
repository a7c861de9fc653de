#!/bin/bash
# A/B of library variants built into build/*.so (python paper_2004_07484_b200/build.py --out=build/x.so -D...):
# per-kernel times of a C3 frame for each, then the GPU parity suite on the ones named in AB_TEST.
# usage: gpurun -- bash scripts/ab_variants.sh "base xu" "xu"
mkdir -p gpurun_out
for v in $1; do
  echo "=== $v"
  SS_B200_LIB=$PWD/build/$v.so QT_STEPS=20 python scripts/quick_time.py 2>&1 | grep -v "^status" | tee gpurun_out/ab_$v.txt
done
for v in $2; do
  echo "=== pytest $v"
  SS_B200_LIB=$PWD/build/$v.so timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 | tee gpurun_out/ab_pytest_$v.txt
done
