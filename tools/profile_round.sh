#!/bin/bash
# One round's measurement set for a config, under gpurun from the repo root
# (B200_PROFILING.md: plain run first, then the launch list, then one --set full capture):
#   bash tools/profile_round.sh TAG CONFIG [KERNEL_REGEX]
#   -> gpurun_out/TAG_bench_CONFIG.json   bench line (cpu_baseline + e2e)
#      gpurun_out/TAG_launches_CONFIG.csv ncu launch list (gpu__time_duration.sum, cold, serialised)
#      gpurun_out/TAG_CONFIG.ncu-rep      ncu --set full of the trace (+ march) kernels
set -u
TAG=$1; CFG=$2; KRE=${3:-regex:k_trace|k_march}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python bench.py --config $CFG --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_${CFG}.json 2> gpurun_out/${TAG}_bench_${CFG}.err
echo "bench rc=$?"; cat gpurun_out/${TAG}_bench_${CFG}.json
# ncu cannot profile kernel nodes of graphs with conditional nodes: profile the host step loop
# (the same kernels, ordinary launches)
CMD="env DPR_STEP_LOOP=host python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_${CFG}.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k "$KRE" -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-3} \
  -o gpurun_out/${TAG}_${CFG} $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
