#!/bin/bash
# Usage (under gpurun, from the repo root): bash tools/gpu_check.sh [tests] [bench] [launches] [full]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
for what in "$@"; do
  case $what in
    tests) timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log;;
    smoke) python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log;;
    bench) timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err;;
    benchq) timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err;;
    launches)
      CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
      $CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?";;
    full)
      CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
      $CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_trace -s 2 -c 2 -o gpurun_out/prof_trace $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?";;
  esac
done
