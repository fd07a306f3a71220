# usage: bash tools/ab_env.sh TAG "ENV=1" "" ... : interleaved bench runs under environment settings (REPS, STEPS, CONFIG)
TAG=$1; shift
for rep in $(seq 1 ${REPS:-2}); do
  i=0
  for e in "$@"; do
    i=$((i+1))
    env $e timeout -s KILL 150 python bench.py --config ${CONFIG:-wan14b_720p} --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_${TAG}_${i}_$rep.json 2>/dev/null
    python -c "import json,sys; d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); print(sys.argv[2] or 'default', round(d['ms_attention'],3), round(d['ms_quantize'],3), d['redo_items'], d['clocks']['sm_mhz'])" gpurun_out/ab_${TAG}_${i}_$rep.json "$e"
  done
done
