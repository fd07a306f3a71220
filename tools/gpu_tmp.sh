timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_r1v.json 2> gpurun_out/bench_r1v.err
