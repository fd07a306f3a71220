# usage: bash tools/gpu_dev.sh TAG  (gpu tests, bench, trace of the attention kernel)
TAG=${1:-x}
timeout -s KILL 400 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 120 > gpurun_out/tests_$TAG.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_$TAG.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout -s KILL 120 python tools/trace_attn.py c2 > gpurun_out/trace_$TAG.txt 2>&1
