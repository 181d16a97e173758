# Full evidence set of a round (run from the repo root under gpurun, one GPU):
#   bench lines for every workload + the reference arm (run_final.sh), the ncu launch list,
#   full captures of k_gemm / k_pack and the tensor-pipe pass (run_ncu.sh), and the 8-rank
#   shared-GPU functional runs (run_shared.sh).  TAG names the round (default r02).
#   Then, here: python profiles/summarize_ncu.py TAG gpurun_out; python profiles/sass_evidence.py TAG
set -u
TAG=${1:-r02}
timeout 3000 bash profiles/run_final.sh gpurun_out/final > gpurun_out/final_rc.log 2>&1
timeout 1500 bash profiles/run_ncu.sh $TAG > gpurun_out/ncu_rc.log 2>&1
timeout 1500 bash profiles/run_shared.sh gpurun_out/shared 8 > gpurun_out/shared_rc.log 2>&1
cat gpurun_out/final_rc.log gpurun_out/ncu_rc.log gpurun_out/shared_rc.log
