for c in 1 2 4; do
timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-chunk $c > gpurun_out/e2e_c$c.json 2>/dev/null
python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], d['e2e']['ms_per_step'], d['ms_per_step'])" gpurun_out/e2e_c$c.json $c >> gpurun_out/e2e_chunks2.txt
done
