#!/bin/bash
# Round evidence run on the B200 box (under gpurun): bench line, 64-view single-GPU anchor for the scaling curve,
# ncu launch list of the bench command, one ncu --set full capture of every kernel of a C3 frame, sanitizer runs.
# Usage: bash scripts/gpu_evidence.sh <tag>      (outputs under gpurun_out/<tag>_*)
tag=${1:-r02}
out=gpurun_out
python bench.py --steps 200 --warmup 20 > $out/${tag}_bench.json 2> $out/${tag}_bench.err
python bench.py --impl reference --steps 1 --warmup 0 > $out/${tag}_bench_reference.json 2>> $out/${tag}_bench.err
python bench.py --steps 20 --warmup 3 --views-per-rank 64 --no-cpu-baseline > $out/${tag}_bench_c4_64views_n1.json 2>> $out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/${tag}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/${tag}_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_' -s 11 -c 11 -o $out/${tag}_full \
    python scripts/quick_time.py > $out/${tag}_full.log 2>&1
# tracked exports of the capture: every raw metric per kernel, the compact per-kernel table + the JSON bench.py
# reads (profiles/ncu_kernels.json), and the per-source-line instruction / stall table of the raster kernel
ncu -i $out/${tag}_full.ncu-rep --page raw --csv > $out/${tag}_ncu_raw_all_metrics.csv 2>/dev/null
python scripts/ncu_extract.py $out/${tag}_ncu_raw_all_metrics.csv $out/${tag}_kernels.csv $out/${tag}_ncu_kernels.json > /dev/null
ncu -i $out/${tag}_full.ncu-rep --page source --csv --print-source cuda,sass > $out/${tag}_src.csv 2>/dev/null
python scripts/ncu_stalls.py $out/${tag}_src.csv k_raster 45 > $out/${tag}_raster_stalls.txt 2>&1
python scripts/launch_shares.py $out/${tag}_launches.csv > $out/${tag}_launch_shares.txt 2>&1
python scripts/run_config.py --count 10000000 --width 1920 --height 1080 --d 16 --k 32 --tau 0.01 > $out/${tag}_c5.log 2>&1
SAN="tests/test_gpu_parity.py::test_golden_forward tests/test_gpu_parity.py::test_golden_backward tests/test_gpu_fuzz.py tests/test_gpu_api.py::test_early_stop_bound_and_chunk_sizes tests/test_gpu_api.py::test_compact_gradient_records_device_array_and_mapped_host_array"
compute-sanitizer --tool memcheck --error-exitcode 1 python -m pytest $SAN -x -q > $out/${tag}_sanitizer_memcheck.log 2>&1
compute-sanitizer --tool racecheck --error-exitcode 1 python -m pytest tests/test_gpu_parity.py::test_golden_forward tests/test_gpu_parity.py::test_golden_backward -x -q > $out/${tag}_sanitizer_racecheck.log 2>&1
compute-sanitizer --tool synccheck --error-exitcode 1 python -m pytest tests/test_gpu_parity.py::test_golden_forward tests/test_gpu_parity.py::test_golden_backward -x -q > $out/${tag}_sanitizer_synccheck.log 2>&1
tail -n 3 $out/${tag}_sanitizer_memcheck.log $out/${tag}_sanitizer_racecheck.log $out/${tag}_sanitizer_synccheck.log
