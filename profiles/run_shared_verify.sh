out=gpurun_out/shared_v
mkdir -p $out
port=29600
for np in 2 4 8; do
 for ex in p2p nccl u32; do
  port=$((port + 1))
  MHG_BENCH_SHARED_GPU=1 MHG_EXCHANGE=$ex timeout 600 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node $np --master-addr 127.0.0.1 --master-port $port bench.py --gpus $np \
      --workload cfg2 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $out/cfg2_${np}_${ex}.log 2> $out/cfg2_${np}_${ex}.err
  echo "cfg2 $np $ex rc=$? $(python -c "import json,sys; d=json.loads(open('$out/cfg2_${np}_${ex}.log').read().strip().splitlines()[-1]); print(d['verified'], d['exchange']['mode'])" 2>&1 | tail -1)"
 done
done
port=29650
MHG_BENCH_SHARED_GPU=1 MHG_EXCHANGE=p2p timeout 900 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node 8 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 8 \
      --workload ns16k --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $out/ns16k_8_p2p.log 2> $out/ns16k_8_p2p.err
echo "ns16k 8 p2p rc=$? $(python -c "import json,sys; d=json.loads(open('$out/ns16k_8_p2p.log').read().strip().splitlines()[-1]); print(d['verified'], d['exchange']['mode'])" 2>&1 | tail -1)"
port=29660
MHG_BENCH_FAIL_P2P_CHECK=1 MHG_BENCH_SHARED_GPU=1 MHG_EXCHANGE=p2p timeout 600 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 \
      --workload cfg2 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $out/cfg2_4_p2pfail.log 2> $out/cfg2_4_p2pfail.err
echo "cfg2 4 p2p->nccl (forced) rc=$? $(python -c "import json,sys; d=json.loads(open('$out/cfg2_4_p2pfail.log').read().strip().splitlines()[-1]); print(d['verified'], d['exchange']['mode'], d['exchange']['note'])" 2>&1 | tail -1)"
