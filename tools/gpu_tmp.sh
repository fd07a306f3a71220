REPS=3 STEPS=20 bash tools/ab.sh ldb libfpsa.so libfpsa_ldb.so > gpurun_out/ab_ldb.txt 2>&1
