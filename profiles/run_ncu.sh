#!/bin/bash
# ncu evidence for the bench workload (run under gpurun, 1 GPU).
# 1) plain run must exit 0; 2) launch list (per-kernel device time, serialized,
# cold-cache: compare SHARES); 3) one full capture of each hot kernel.
set -u
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
TAG=${1:-r01}
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 1 \
    -o gpurun_out/${TAG}_gemm_full $CMD > gpurun_out/${TAG}_ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pack -s 4 -c 2 \
    -o gpurun_out/${TAG}_pack_full $CMD > gpurun_out/${TAG}_ncu_pack.log 2>&1
# tensor-pipe evidence for the GEMM: UTCIMMA sub-pipe active cycles / instructions, TMEM
# bytes read by LDTM (epilogue drains), elapsed cycles
TP="sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_imma.sum,sm__mem_tensor_reads_op_ldt.sum,sm__cycles_elapsed.avg,gpu__time_duration.sum"
ncu --metrics $TP --clock-control none -k regex:k_gemm -s 2 -c 1 --csv \
    --log-file gpurun_out/${TAG}_tensor_pipe.csv $CMD > gpurun_out/${TAG}_ncu_tp.log 2>&1
echo "ncu done"
