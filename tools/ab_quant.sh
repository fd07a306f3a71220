# usage: bash tools/ab_quant.sh TAG lib1 lib2 ... : interleaved tools/bench_quant.py runs of in-tree library variants
TAG=$1; shift
for rep in $(seq 1 ${REPS:-2}); do
  for lib in "$@"; do
    echo -n "$lib "
    FPSA_LIB=$lib timeout -s KILL 120 python tools/bench_quant.py 2>&1 | tail -1
  done
done | tee gpurun_out/abq_$TAG.txt
