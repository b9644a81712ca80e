#!/bin/bash
# Time opbench for several libdg variants / env settings on one GPU box.
#   tools/variants.sh OPS SCALE "label:lib:ENV=..;ENV2=.." ...
OPS=$1; SCALE=$2; shift 2
for spec in "$@"; do
  IFS=: read -r label lib envs <<< "$spec"
  [ -n "$lib" ] && export DG_LIB_PATH=$lib || unset DG_LIB_PATH
  echo "== $label"
  env $(echo "$envs" | tr ';' ' ') python tools/opbench.py --ops $OPS --scale $SCALE --reps 10 2>&1 | \
    python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(f\"  {d['op']:10s} {d['ms']:9.3f} ms  {d['frac_hbm']:.3f}\")
    except Exception: print('  ', l.strip()[:200])"
done
