timeout -s KILL 120 python tools/debug_pad8.py > gpurun_out/pad8b.txt 2>&1
timeout -s KILL 400 python -m pytest tests/test_gpu_attention.py -q -s -p no:cacheprovider --timeout 100 -k "emulation or golden or redo or full_size" > gpurun_out/tests_attn_r2v.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_attn_r2v.txt
