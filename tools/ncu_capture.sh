#!/bin/bash
# ncu --set full of one workload's kernels on the GPU box, exported there to CSV (the .ncu-rep
# files exceed gpurun's return cap):
#   bash tools/ncu_capture.sh TAG CFG KREGEX SKIP COUNT "K1 K2" [cmd...]
#   -> gpurun_out/TAG_raw_CFG.csv (raw page), gpurun_out/TAG_src_CFG_K.csv per kernel K (source
#      page, cuda + sass, for tools/ncu_lines.py)
TAG=$1; CFG=$2; KRE=$3; SKIP=$4; COUNT=$5; SRCK=$6; shift 6
CMD=${@:-python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e}
mkdir -p gpurun_out
# kernel nodes of CUDA graphs with conditional nodes cannot be profiled: the step loop runs on
# the host here (the same kernels as the device-driven loop, ordinary launches)
export DPR_STEP_LOOP=host
$CMD > gpurun_out/plain_${CFG}.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k "$KRE" -s $SKIP -c $COUNT -o /tmp/${TAG}_${CFG} $CMD > gpurun_out/ncu_${CFG}.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/${TAG}_${CFG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw_${CFG}.csv 2>/dev/null
for K in $SRCK; do
  ncu -i /tmp/${TAG}_${CFG}.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:$K > gpurun_out/${TAG}_src_${CFG}_${K}.csv 2>/dev/null
done
ncu -i /tmp/${TAG}_${CFG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details_${CFG}.csv 2>/dev/null
ls -la gpurun_out/${TAG}_*_${CFG}.csv
