# usage: bash tools/ab_quant_env.sh TAG "ENV1" "ENV2" ... : interleaved tools/bench_quant.py runs under env settings ("-" = none)
TAG=$1; shift
for rep in $(seq 1 ${REPS:-2}); do
  for e in "$@"; do
    echo -n "$e "
    if [ "$e" = "-" ]; then timeout -s KILL 120 python tools/bench_quant.py 2>&1 | tail -1
    else env $e timeout -s KILL 120 python tools/bench_quant.py 2>&1 | tail -1; fi
  done
done | tee gpurun_out/abqe_$TAG.txt
