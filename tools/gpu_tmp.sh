for i in 1 2 3 4 5; do
timeout -s KILL 300 python bench.py --no-cpu > gpurun_out/rep_$i.json 2>/dev/null
python -c "import json,sys; d=json.load(open(sys.argv[1])); print('run', sys.argv[2], 'step', round(d['ms_per_step'],3), 'attn', round(d['ms_attention'],3), 'quant', round(d['ms_quantize'],3), 'TF', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'e2e_ms', round(d['e2e']['ms_per_step'],2), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" gpurun_out/rep_$i.json $i >> gpurun_out/bench_repeats.txt
done
