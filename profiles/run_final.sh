#!/bin/bash
# Full bench lines for every BASELINE workload + the reference arm (1 GPU).
# usage: profiles/run_final.sh OUTDIR
out=${1:-gpurun_out/final}
mkdir -p $out
for w in ns16k cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w > $out/$w.log 2> $out/$w.err
  echo "$w rc=$?"
done
timeout 900 python bench.py --impl reference > $out/ref.log 2> $out/ref.err
echo "ref rc=$?"
