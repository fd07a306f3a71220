# usage: bash tools/gpu_prof.sh TAG [bench args]  (ncu --set full of one attention launch)
TAG=${1:-x}; shift
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fpsa_attn -s 2 -c 1 -o gpurun_out/attn_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/ncu_attn_$TAG.out 2>&1
