timeout -s KILL 500 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 200 > gpurun_out/tests_r1r.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_r1r.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1r.json 2> gpurun_out/bench_r1r.err
timeout -s KILL 300 python tools/sweep.py --csv gpurun_out/sweep_c4_r1r.csv > gpurun_out/sweep_r1r.json 2> gpurun_out/sweep_r1r.err
