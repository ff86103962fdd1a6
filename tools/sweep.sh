#!/bin/bash
# Build tuning variants on the GPU box and bench each (device-resident leg only).
# Usage: bash tools/sweep.sh "NAME:-DFOO=1 -DBAR=2" "NAME2:..." ...
mkdir -p gpurun_out/sweep
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  python paper_2407_00179_b200/build.py --force --out=/tmp/libdpr_$name.so $defs > gpurun_out/sweep/$name.build 2>&1 || { echo "$name BUILD FAILED"; continue; }
  DPR_LIB=/tmp/libdpr_$name.so python bench.py $SWEEP_ARGS --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sweep/$name.json 2> gpurun_out/sweep/$name.err
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
