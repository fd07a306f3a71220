REPS=3 STEPS=20 bash tools/ab.sh poly3 libfpsa.so libfpsa_p6.so libfpsa_p8.so > gpurun_out/ab_poly3_pp.txt 2>&1
