TAG=${1:-x}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 14 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"quant|amax" -s 2 -c 2 -o gpurun_out/quant_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_quant_$TAG.out 2>&1
