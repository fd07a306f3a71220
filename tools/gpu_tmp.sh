timeout -s KILL 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r3v.txt 2>&1; echo "EXIT $?" >> gpurun_out/smoke_r3v.txt
timeout -s KILL 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 200 > gpurun_out/tests_r3v.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_r3v.txt
timeout -s KILL 300 python bench.py > gpurun_out/bench_r3v.json 2> gpurun_out/bench_r3v.err
