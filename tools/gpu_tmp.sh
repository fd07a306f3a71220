timeout -s KILL 60 tools/probes/mma2_rate > gpurun_out/mma2_rate.txt 2>&1; echo "EXIT $?" >> gpurun_out/mma2_rate.txt
