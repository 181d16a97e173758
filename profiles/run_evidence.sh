# Full evidence set of a round (run from the repo root under gpurun): bench lines for every
# workload + the reference arm, the ncu launch list and full captures, the k_widen16 capture.
set -u
bash profiles/run_final.sh gpurun_out/final > gpurun_out/final_rc.log 2>&1
bash profiles/run_ncu.sh r01l > gpurun_out/ncu_rc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_widen16 -c 1 -o gpurun_out/r01l_widen_full python profiles/upload_wire.py 16384 1 > gpurun_out/ncu_widen.log 2>&1
cat gpurun_out/final_rc.log gpurun_out/ncu_rc.log
