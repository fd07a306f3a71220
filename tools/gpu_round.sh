# usage: bash tools/gpu_round.sh TAG   (runs gpu tests, bench, launch list, ncu of attention + quantiser)
TAG=${1:-x}
timeout -s KILL 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 300 > gpurun_out/tests_$TAG.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_$TAG.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fpsa_attn|quant_tma|quant_ldg|chan_amax" -c 12 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fpsa_attn -s 2 -c 1 -o gpurun_out/attn_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_attn_$TAG.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quant_tma -s 1 -c 1 -o gpurun_out/quant_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_quant_$TAG.out 2>&1
