# usage: bash tools/gpu_evidence.sh TAG  (bench line, ncu launch list, ncu --set full of attention + quantiser, summaries)
TAG=${1:-x}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fpsa_attn|quant_tma|chan_amax" -c 12 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fpsa_attn -s 2 -c 1 -o gpurun_out/attn_$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_attn_$TAG.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quant_tma -s 1 -c 1 -o gpurun_out/quant_$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_quant_$TAG.out 2>&1
python tools/ncu_summary.py gpurun_out/attn_$TAG.ncu-rep --json gpurun_out/attn_ncu_$TAG.json > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/quant_$TAG.ncu-rep --json gpurun_out/quant_ncu_$TAG.json > /dev/null 2>&1
ncu -i gpurun_out/attn_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/attn_src_$TAG.csv 2>/dev/null
python tools/sass_stalls.py gpurun_out/attn_src_$TAG.csv --top 40 > gpurun_out/attn_stalls_$TAG.txt 2>&1
rm -f gpurun_out/attn_src_$TAG.csv
