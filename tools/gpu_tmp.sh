timeout -s KILL 400 python -m pytest tests/test_bench_contract.py -q -p no:cacheprovider > gpurun_out/tests_bench_r3h.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_bench_r3h.txt
