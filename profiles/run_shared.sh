#!/bin/bash
# N > 1 functional runs of bench.py with every rank on ONE GPU (MHG_BENCH_SHARED_GPU=1:
# gloo collectives, host-staged; never a measurement -- the ranks share one device).
# Exercises both exchanges (copy-engine pulls over IPC, packed broadcasts) at the
# north-star size and at cfg5.  usage: profiles/run_shared.sh OUTDIR [NPROC]
out=${1:-gpurun_out/shared}
np=${2:-8}
mkdir -p $out
port=29533
for w in ns16k cfg5; do
  for ex in p2p nccl; do
    port=$((port + 1))
    MHG_BENCH_SHARED_GPU=1 MHG_EXCHANGE=$ex timeout 900 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node $np --master-addr 127.0.0.1 --master-port $port bench.py --gpus $np \
      --workload $w --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $out/${w}_${ex}.log 2> $out/${w}_${ex}.err
    echo "$w $ex rc=$?"
  done
done
