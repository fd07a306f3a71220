timeout -s KILL 60 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1y.txt 2>&1; echo "EXIT $?" >> gpurun_out/smoke_r1y.txt
timeout -s KILL 400 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 120 > gpurun_out/tests_r1y.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_r1y.txt
timeout -s KILL 400 python bench.py > gpurun_out/bench_r1y.json 2> gpurun_out/bench_r1y.err
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r1y.json 2> gpurun_out/bench_ref_r1y.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_r1y.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fpsa_attn -s 2 -c 1 -o gpurun_out/attn_r1y python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_attn_r1y.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quant_tma -s 1 -c 1 -o gpurun_out/quant_r1y python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_quant_r1y.out 2>&1
timeout -s KILL 300 python tools/sweep.py --csv gpurun_out/sweep_c4_r1y.csv > gpurun_out/sweep_r1y.json 2> gpurun_out/sweep_r1y.err
timeout -s KILL 200 python bench.py --config wan13b_480p --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c1_r1y.json 2>&1
timeout -s KILL 200 python bench.py --config wan14b_720p_w333 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_w333_r1y.json 2>&1
timeout -s KILL 200 python bench.py --config hunyuan_720p --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3_r1y.json 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r1y.txt
