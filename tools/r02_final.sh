#!/bin/bash
# Round-2 end-of-round evidence on one B200 (run under gpurun): GPU tests,
# smoke, the default bench line and the reference arm -> gpurun_out/final/
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final/gpu_tests.txt 2>&1
tail -2 gpurun_out/final/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.txt 2>&1
tail -1 gpurun_out/final/smoke.txt
timeout 900 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err
tail -c 400 gpurun_out/final/bench_default.json
if [ "${REF:-1}" = 1 ]; then
  timeout 1500 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
  tail -c 300 gpurun_out/final/bench_reference.json
fi
