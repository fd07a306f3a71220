timeout -s KILL 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r3q.txt 2>&1; echo "EXIT $?" >> gpurun_out/smoke_r3q.txt
timeout -s KILL 500 python -m pytest tests/test_gpu_attention.py tests/test_gpu_multistep.py -x -q -p no:cacheprovider --timeout 100 > gpurun_out/tests_r3q.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_r3q.txt
REPS=3 STEPS=20 bash tools/ab.sh half libfpsa_r3p.so libfpsa.so > gpurun_out/ab_half.txt 2>&1
