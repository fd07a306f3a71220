# quantiser rewrite (libfpsa_nq.so): bit-exactness tests + timing; ncu source page of the split-issue attention variant
FPSA_LIB=libfpsa_nq.so timeout -s KILL 600 python -m pytest tests/test_gpu_quant.py tests/test_gpu_dropin.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/tests_nq.txt 2>&1
REPS=3 bash tools/ab_quant.sh nq libfpsa.so libfpsa_nq.so > /dev/null 2>&1
FPSA_LIB=libfpsa_e2.so timeout 400 ncu --set full --clock-control none --import-source on -k regex:fpsa_attn -s 2 -c 1 -o gpurun_out/attn_e2 -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_attn_e2.out 2>&1
ncu -i gpurun_out/attn_e2.ncu-rep --page source --csv --print-source sass > gpurun_out/attn_src_e2.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/attn_e2.ncu-rep --json gpurun_out/attn_ncu_e2.json > /dev/null 2>&1
