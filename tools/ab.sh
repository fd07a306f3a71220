# usage: bash tools/ab.sh TAG lib1 lib2 ... : interleaved bench runs of in-tree library variants (REPS, STEPS env)
TAG=$1; shift
for rep in $(seq 1 ${REPS:-2}); do
  for lib in "$@"; do
    FPSA_LIB=$lib timeout -s KILL 120 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_${TAG}_${lib}_$rep.json 2>/dev/null
    python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], d['ms_attention'], d['ms_quantize'], d['redo_items'], d['clocks']['sm_mhz'])" gpurun_out/ab_${TAG}_${lib}_$rep.json $lib
  done
done
