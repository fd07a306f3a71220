timeout -s KILL 300 python -m pytest tests/test_gpu_multistep.py -x -q -p no:cacheprovider --timeout 100 > gpurun_out/tests_ms_r2t.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_ms_r2t.txt
