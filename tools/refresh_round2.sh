#!/bin/bash
# Round-2 measurement evidence (run under gpurun, one GPU, ~20 min):
#   bash tools/refresh_round2.sh  -> gpurun_out/r2/*
set -x
O=gpurun_out/r2
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --workload c3 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --workload splom --steps 10 > $O/bench_splom.json 2> $O/bench_splom.err
python bench.py --workload sweep > $O/bench_sweep.json 2> $O/bench_sweep.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --impl reference --workload splom --steps 3 --warmup 3 > $O/bench_ref_splom.json 2> $O/bench_ref_splom.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -c 800 --csv --log-file $O/launches_bench_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-splom > $O/ncu_bench_c2.log 2>&1
PROF_ITERS=3 ncu --metrics $M --clock-control none --csv --log-file $O/launches_iter_c3.csv \
    python tools/prof_driver.py iter3 > $O/ncu_iter_c3.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file $O/launches_integral.csv \
    python tools/prof_driver.py integral --big > $O/ncu_int.log 2>&1
PROF_PLOTS=32 PROF_ITERS=10 ncu --metrics $M --clock-control none --csv --log-file $O/launches_splom.csv \
    python tools/prof_driver.py splom > $O/ncu_splom.log 2>&1
ATOM=lts__t_requests_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,smsp__inst_executed_op_global_red.sum,lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_red.sum
PROF_ITERS=3 ncu --set full --import-source on --clock-control none --metrics $ATOM \
    -k regex:"splat|smooth|lines|chains|write_kernel|sample_f32" --launch-skip 0 -c 9 \
    -o $O/full_iter_c2 python tools/prof_driver.py iter > $O/ncu_full_c2.log 2>&1
PROF_ITERS=3 ncu --set full --import-source on --clock-control none --metrics $ATOM \
    -k regex:"splat_f32|sample_f32|smooth|write_kernel|chains" --launch-skip 0 -c 8 \
    -o $O/full_iter_c3 python tools/prof_driver.py iter3 > $O/ncu_full_c3.log 2>&1
PROF_PLOTS=32 PROF_ITERS=3 ncu --set full --import-source on --clock-control none \
    -k regex:"move_bulk|write_kernel|smooth_v|smooth_h|chains" --launch-skip 10 -c 5 \
    -o $O/full_splom python tools/prof_driver.py splom > $O/ncu_full_splom.log 2>&1
ls -la $O
