FPSA_TRACE_LIB=libfpsa_trace_pp4.so timeout -s KILL 120 python tools/trace_attn.py c2 > gpurun_out/trace_pp4.txt 2>&1
