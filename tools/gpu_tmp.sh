timeout -s KILL 60 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r3d.txt 2>&1; echo "EXIT $?" >> gpurun_out/smoke_r3d.txt
if grep -q "smoke ok" gpurun_out/smoke_r3d.txt; then
timeout -s KILL 400 python -m pytest tests/test_gpu_attention.py tests/test_gpu_multistep.py -x -q -p no:cacheprovider --timeout 60 > gpurun_out/tests_r3d.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_r3d.txt
bash tools/ab.sh trio libfpsa_pp1.so libfpsa.so > gpurun_out/ab_trio.txt 2>&1
timeout -s KILL 120 python tools/trace_attn.py c2 > gpurun_out/trace_r3d.txt 2>&1
fi
