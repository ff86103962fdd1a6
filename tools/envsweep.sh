#!/bin/bash
# Bench the default library under different environment settings.
# Usage: bash tools/envsweep.sh "NAME:VAR=val VAR2=val" ...
mkdir -p gpurun_out/sweep
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  env $envs python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sweep/$name.json 2> gpurun_out/sweep/$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    j = json.load(open(f"gpurun_out/sweep/{n}.json"))
    w = j["work_rank0"]
    print(f"{n:14s} {j['value']/1e6:8.1f} Mray/s step {j['ms_per_step']:6.2f} frame {j['ms_per_frame']:6.2f} build {j['ms_build']:5.2f} "
          f"{j['roofline']['kernel']} {j['roofline']['avg_launch_ms']:6.2f} other {j['roofline']['other_kernel_ms_per_step']:6.2f} "
          f"nodes p/o {w['k_trace_path']['nodes_per_ray']:.1f}/{w['k_trace_occl']['nodes_per_ray']:.1f} tris p/o {w['k_trace_path']['tris_per_ray']:.1f}/{w['k_trace_occl']['tris_per_ray']:.1f}")
except Exception as e:
    print(n, "FAILED", e)
PY
done
