for i in 1 2; do
for lib in main tmem256; do
if [ $lib = main ]; then unset GFM_LIB_PATH; else export GFM_LIB_PATH=paper_2406_12909_b200/_lib/$lib/libgfm_b200.so; fi
for c in c2 c3; do
python bench.py --config $c --steps 30 --warmup 5 --cpu-sample-s 0.5 --no-nested 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $c', round(d['value']), round(d['ms_per_step'], 4), d['roofline']['launch_ms'])"
done; done; done
