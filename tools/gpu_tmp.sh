timeout -s KILL 300 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_racecheck.txt 2>&1; echo "EXIT $?" >> gpurun_out/sanitizer_racecheck.txt
timeout -s KILL 300 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_memcheck.txt 2>&1; echo "EXIT $?" >> gpurun_out/sanitizer_memcheck.txt
timeout -s KILL 300 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 200 > gpurun_out/tests_r2e.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_r2e.txt
timeout -s KILL 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err
