#!/bin/bash
# One GPU call covering a round's evidence (run from the repo root under gpurun):
#   tools/gpu_round.sh [tests|bench|launches|full|all]...
# tests    -> gpurun_out/pytest.log, parity.json (achieved errors), smoke.log
# bench    -> gpurun_out/bench.json (+ bench.err)
# small    -> gpurun_out/small_<cfg>_g<0|1>.json (cfg2 / cfg1 lines, device Arnoldi scalars on / off)
# launches -> gpurun_out/launches.csv (ncu launch list of one bench step)
# full     -> gpurun_out/helm.ncu-rep, expl.ncu-rep (ncu --set full at cfg4 size:
#             the first kernels of one GMRES solve; the explicit operator)
# Each step runs only after the previous command exited; a number printed
# under ncu is never a bench value.
mkdir -p gpurun_out
steps=${*:-all}
has() { [[ " $steps " == *" $1 "* || " $steps " == *" all "* ]]; }
if has tests; then
  DG_PARITY_LOG=gpurun_out/parity.json timeout 2400 python -m pytest tests -m gpu -x -q \
    > gpurun_out/pytest.log 2>&1
  echo "pytest rc $?"; tail -3 gpurun_out/pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  echo "smoke rc $?"; tail -2 gpurun_out/smoke.log
fi
if has bench; then
  timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc $?"; tail -c 600 gpurun_out/bench.json
fi
if has small; then
  for w in cfg2 cfg1; do
    for gm in 1 0; do
      DG_DEVARN=$gm timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline \
        > gpurun_out/small_${w}_g$gm.json 2> gpurun_out/small_${w}_g$gm.err
      echo "small $w devarn=$gm rc $?"; tail -c 300 gpurun_out/small_${w}_g$gm.json
    done
  done
fi
if has launches; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 600 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launches.log 2>&1
  echo "launches rc $?"
fi
if has full; then
  timeout 1200 ncu --set full --clock-control none --import-source on -s 0 -c 10 -f \
    -o gpurun_out/helm python tools/opbench.py --case cfg4 --scale 1.0 --ops gmres --reps 1 \
    > gpurun_out/ncu_helm.log 2>&1
  echo "full helm rc $?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"xelem_kernel" -s 1 -c 1 -f \
    -o gpurun_out/expl python tools/opbench.py --case cfg4 --scale 1.0 --ops explicit --reps 1 \
    > gpurun_out/ncu_expl.log 2>&1
  echo "full expl rc $?"
fi
# summaries on the box (gpurun copies back <= 64 MiB): launch list, per-kernel
# tables, DRAM traffic vs algorithmic bytes, opcode mix of every captured
# launch; reports larger than 24 MB are dropped after summarising
if [ -f gpurun_out/launches.csv ]; then
  python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches.md
fi
for r in helm expl; do
  [ -f gpurun_out/$r.ncu-rep ] || continue
  python tools/ncu_summary.py full gpurun_out/$r.ncu-rep > gpurun_out/$r.kernels.md
  n=$(ncu -i gpurun_out/$r.ncu-rep --page raw --csv --metrics gpu__time_duration.sum 2>/dev/null | tail -n +3 | wc -l)
  for ((i = 0; i < n; i++)); do
    python tools/ncu_opmix.py gpurun_out/$r.ncu-rep $i 30 > gpurun_out/$r.opmix.$i.txt
  done
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv
done
[ -f gpurun_out/helm.ncu-rep ] && python tools/traffic_json.py gpurun_out/helm.ncu-rep \
  gpurun_out/expl.ncu-rep > gpurun_out/traffic.json
find gpurun_out -name "*.ncu-rep" -size +24M -delete
gzip -f gpurun_out/launches.csv 2>/dev/null
du -sh gpurun_out
