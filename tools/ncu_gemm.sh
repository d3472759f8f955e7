#!/bin/bash
# ncu --set full of selected tcgen05 GEMM launches in the eager C3 step.
# Usage (under gpurun): tools/ncu_gemm.sh <config> <skip> <count> <tag>
cfg=$1; skip=$2; cnt=$3; tag=$4
mkdir -p gpurun_out
python tools/step_once.py --config $cfg --steps 1 > gpurun_out/g_plain_$tag.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm --launch-skip $skip \
    -c $cnt -o /tmp/g_$tag -f python tools/step_once.py --config $cfg --steps 1 \
    > gpurun_out/g_$tag.log 2>&1
python tools/ncu_raw.py /tmp/g_$tag.ncu-rep > gpurun_out/g_$tag.txt 2>&1
ncu -i /tmp/g_$tag.ncu-rep --page raw --csv > gpurun_out/g_$tag.raw.csv 2>/dev/null
ncu -i /tmp/g_$tag.ncu-rep --page source --csv > gpurun_out/g_$tag.src.csv 2>/dev/null
