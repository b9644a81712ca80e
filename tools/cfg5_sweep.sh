#!/bin/bash
# Operator microbenchmark (BASELINE configs[4]): explicit-operator and
# Helmholtz-apply throughput on the periodic cfg5 box at r = 2..6, ~1e8 DoF,
# with the fp64 FMA peak measured first (tools/dfma_peak).
#   tools/cfg5_sweep.sh [scale] > gpurun_out/cfg5.jsonl
SCALE=${1:-1.0}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
[ -x $ROOT/tools/dfma_peak ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
  -o $ROOT/tools/dfma_peak $ROOT/tools/dfma_peak.cu
PK=$($ROOT/tools/dfma_peak)
echo "$PK"
export DG_FP64_TFLOPS=$(python -c "import json,sys; print(json.loads(sys.argv[1])['dfma_tflops'])" "$PK")
for r in 2 3 4 5 6; do
  python $ROOT/tools/opbench.py --case cfg5_r$r --scale $SCALE --reps 10 --ops explicit,helmholtz
done
