#!/bin/bash
# Round-2 ncu captures (run under gpurun, one GPU):
#   bash tools/prof_round2.sh  -> gpurun_out/prof2/*
O=gpurun_out/prof2
mkdir -p $O
ATOM=lts__t_requests_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,smsp__inst_executed_op_global_red.sum,lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_red.sum
# C2 iteration kernels, full set + source + the splat's atomic counters
PROF_ITERS=2 ncu --set full --import-source on --clock-control none --metrics $ATOM \
    -k regex:"splat|smooth|lines|chains|write_kernel|sample_f32" --launch-skip 0 -c 9 \
    -o $O/full_iter_c2 python tools/prof_driver.py iter > $O/ncu_full_c2.log 2>&1
# C3: the move + splat and the first splat (atomics at 16M points)
PROF_ITERS=1 ncu --set full --import-source on --clock-control none --metrics $ATOM \
    -k regex:"splat_f32|sample_f32|place_points|unpermute" -c 4 \
    -o $O/full_iter_c3 python tools/prof_driver.py iter3 > $O/ncu_full_c3.log 2>&1
ls -la $O
