mkdir -p gpurun_out
python tools/gemm_one.py wgrad 1 51200 2560 0 512 > gpurun_out/wg_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o /tmp/wg -f python tools/gemm_one.py wgrad 1 51200 2560 0 512 > gpurun_out/wg_ncu.log 2>&1
python tools/ncu_raw.py /tmp/wg.ncu-rep > gpurun_out/wg.txt 2>&1
ncu -i /tmp/wg.ncu-rep --page raw --csv > gpurun_out/wg.raw.csv 2>/dev/null
ncu -i /tmp/wg.ncu-rep --page source --csv > gpurun_out/wg.src.csv 2>/dev/null
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-sample-s 2 > gpurun_out/bench.log 2>&1
timeout 400 python bench.py --config c3 --steps 10 --warmup 3 --cpu-sample-s 2 > gpurun_out/bench_c3.log 2>&1
