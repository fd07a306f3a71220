# usage: bash tools/gpu_quick.sh TAG  (gpu tests + bench only)
TAG=${1:-x}
timeout -s KILL 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 300 > gpurun_out/tests_$TAG.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_$TAG.txt
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
