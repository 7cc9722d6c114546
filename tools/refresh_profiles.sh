#!/bin/bash
# Re-measure every committed profile of this round (run under gpurun; ~10 min):
#   bash tools/refresh_profiles.sh   -> gpurun_out/prof/*
set -x
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --workload c3 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --workload splom > $O/bench_splom.json 2> $O/bench_splom.err
python bench.py --workload sweep > $O/bench_sweep.json 2> $O/bench_sweep.err
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -c 800 --csv --log-file $O/launches_bench_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench_c2.log 2>&1
PROF_ITERS=3 ncu --metrics $M --clock-control none --csv --log-file $O/launches_iter_c3.csv \
    python tools/prof_driver.py iter3 > $O/ncu_iter_c3.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file $O/launches_integral.csv \
    python tools/prof_driver.py integral --big > $O/ncu_int.log 2>&1
PROF_ITERS=2 ncu --set full --import-source on --clock-control none -k regex:"splat|smooth|lines|chains|write_kernel|sample_f32" \
    --launch-skip 0 -c 8 -o $O/full_iter_c2 python tools/prof_driver.py iter > $O/ncu_full_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"reduce|lines|chains|write_kernel" -c 4 \
    -o $O/full_int4096 python tools/prof_driver.py integral > $O/ncu_full_int.log 2>&1
ls -la $O
