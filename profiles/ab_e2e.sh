#!/bin/bash
# e2e A/B of library builds: bench.py's end-to-end line (pinned host, 3 container sets) per build,
# builds interleaved.  usage: profiles/ab_e2e.sh ROUNDS name=lib ...
rounds=$1; shift
for r in $(seq 1 $rounds); do
  for spec in "$@"; do
    name=${spec%%=*}; lib=${spec#*=}
    MHG_LIB=$lib timeout 300 python bench.py --steps 5 --e2e-steps 20 --no-cpu-baseline > /tmp/ab_e2e.log 2>&1
    python - "$name" "$r" <<'PY'
import json, sys
for l in open("/tmp/ab_e2e.log"):
    if l.startswith("{"):
        d = json.loads(l); e = d["e2e"]
        print(f"round {sys.argv[2]} {sys.argv[1]:6s} e2e {e['ms_per_step']:.2f} ms/step  h2d {e['h2d_bytes_per_step']}  device {d['ms_per_step']:.2f} ms")
PY
  done
done
