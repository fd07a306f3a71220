set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches1.out 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fpsa_attn -s 1 -c 1 -o gpurun_out/attn_full1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_attn1.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quant_tile -s 2 -c 1 -o gpurun_out/quant_full1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_quant1.out 2>&1
ls -la gpurun_out
