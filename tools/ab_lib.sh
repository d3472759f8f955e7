mkdir -p gpurun_out
V=paper_2406_12909_b200/_lib/var/libgfm_b200.so
python tools/gemm_sweep.py 1 > gpurun_out/sw_a.log 2>&1
GFM_LIB_PATH=$V python tools/gemm_sweep.py 1 > gpurun_out/sw_b.log 2>&1
for i in 1 2; do
python bench.py --steps 30 --warmup 5 --cpu-sample-s 0.5 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', d['value'], d['e2e']['value'])" >> gpurun_out/ab.log
GFM_LIB_PATH=$V python bench.py --steps 30 --warmup 5 --cpu-sample-s 0.5 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', d['value'], d['e2e']['value'])" >> gpurun_out/ab.log
done
GFM_LIB_PATH=$V timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/b_tests.log 2>&1
