timeout -s KILL 300 python -m pytest tests/test_gpu_quant.py -x -q -p no:cacheprovider --timeout 100 > gpurun_out/tests_q_r3i.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_q_r3i.txt
REPS=3 bash tools/ab.sh q4 libfpsa_qold.so libfpsa.so > gpurun_out/ab_q4.txt 2>&1
