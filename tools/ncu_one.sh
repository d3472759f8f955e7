#!/bin/bash
# ncu --set full of the first launch whose demangled name matches a regex, in
# the eager bench step.  Usage (under gpurun): tools/ncu_one.sh <config> <tag> <regex> [skip]
cfg=$1; tag=$2; rx=$3; skip=${4:-0}
mkdir -p gpurun_out
python tools/step_once.py --config $cfg --steps 1 > gpurun_out/one_plain_$tag.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$rx" --launch-skip $skip -c 1 -o /tmp/one_$tag -f \
    python tools/step_once.py --config $cfg --steps 1 > gpurun_out/one_$tag.log 2>&1
python tools/ncu_raw.py /tmp/one_$tag.ncu-rep > gpurun_out/one_$tag.txt 2>&1
ncu -i /tmp/one_$tag.ncu-rep --page raw --csv > gpurun_out/one_$tag.raw.csv 2>/dev/null
ncu -i /tmp/one_$tag.ncu-rep --page source --csv > gpurun_out/one_$tag.src.csv 2>/dev/null
