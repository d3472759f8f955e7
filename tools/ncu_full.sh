#!/bin/bash
# Full ncu capture (one launch each) of the named kernels in the eager bench
# step, summarised to text on the box (reps are large; only the text and the
# raw csv come back).  Usage (under gpurun):
#   tools/ncu_full.sh <config> <tag> <kernel-regex>...
cfg=$1; tag=$2; shift 2
mkdir -p gpurun_out
python tools/step_once.py --config $cfg --steps 1 > gpurun_out/full_plain_$tag.log 2>&1 || exit 1
i=0
for k in "$@"; do
  rep=/tmp/full_${tag}_$i
  ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 \
      -o $rep -f python tools/step_once.py --config $cfg --steps 1 \
      > gpurun_out/full_${tag}_$i.log 2>&1
  python tools/ncu_raw.py $rep.ncu-rep > gpurun_out/full_${tag}_$i.txt 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/full_${tag}_$i.raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv > gpurun_out/full_${tag}_$i.src.csv 2>/dev/null
  i=$((i+1))
done
