#!/bin/bash
# A/B two builds of libmhg.so on the same box: alternates processes so clock /
# power drift hits both equally.  usage: ab_builds.sh libA.so libB.so rounds cmd...
A=$1; B=$2; R=$3; shift 3
for r in $(seq 1 $R); do
  for v in A B; do
    lib=$A; [ $v = B ] && lib=$B
    echo "== round $r variant $v"
    MHG_LIB=$lib "$@"
  done
done
