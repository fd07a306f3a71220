timeout -s KILL 60 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2f.txt 2>&1; echo "EXIT $?" >> gpurun_out/smoke_r2f.txt
if grep -q "smoke ok" gpurun_out/smoke_r2f.txt; then
timeout -s KILL 300 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 100 > gpurun_out/tests_r2f.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_r2f.txt
timeout -s KILL 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_r2f.json 2> gpurun_out/bench_r2f.err
timeout -s KILL 120 python tools/trace_attn.py c2 > gpurun_out/trace_r2f.txt 2>&1
fi
