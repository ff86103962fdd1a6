#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run first, then the ncu launch list, then one
# --set full capture of the trace kernels.  Run under gpurun from the repo root.
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python -c "import __graft_entry__ as g; g.build()"
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_trace -s 2 -c 2 -o gpurun_out/prof_trace $CMD > gpurun_out/ncu_full.log 2>&1
echo done
