FPSA_LIB=libfpsa_pp4.so timeout -s KILL 400 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider --timeout 60 > gpurun_out/tests_pp4.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_pp4.txt
REPS=3 STEPS=20 bash tools/ab.sh pp4 libfpsa.so libfpsa_pp4.so > gpurun_out/ab_pp4.txt 2>&1
