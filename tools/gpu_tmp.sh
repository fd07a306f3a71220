timeout -s KILL 300 python -m pytest tests/test_gpu_multistep.py -x -q -p no:cacheprovider --timeout 100 > gpurun_out/tests_ms_r2s.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_ms_r2s.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_r2s.json 2> gpurun_out/bench_r2s.err
