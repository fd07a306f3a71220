timeout -s KILL 300 python -m pytest tests/test_gpu_quant.py -x -q -p no:cacheprovider --timeout 100 > gpurun_out/tests_q_r2r.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_q_r2q.txt
bash tools/ab.sh q3 libfpsa_qold.so libfpsa.so > gpurun_out/ab_q3.txt 2>&1
