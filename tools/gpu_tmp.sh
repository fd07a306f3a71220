REPS=1 STEPS=10 bash tools/ab.sh a2x libfpsa_a2.so libfpsa_a2n.so > gpurun_out/ab_a2x.txt 2>&1
