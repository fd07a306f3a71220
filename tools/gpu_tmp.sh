timeout -s KILL 60 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2o.txt 2>&1; echo "EXIT $?" >> gpurun_out/smoke_r2o.txt
if grep -q "smoke ok" gpurun_out/smoke_r2o.txt; then
timeout -s KILL 400 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 100 > gpurun_out/tests_r2o.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_r2o.txt
timeout -s KILL 300 python bench.py > gpurun_out/bench_r2o.json 2> gpurun_out/bench_r2o.err
fi
