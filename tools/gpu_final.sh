# usage: bash tools/gpu_final.sh TAG  (round-end evidence: tests, bench, launch list, ncu, configs, sweep, trace)
TAG=${1:-x}
timeout -s KILL 60 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; echo "EXIT $?" >> gpurun_out/smoke_$TAG.txt
bash tools/gpu_round.sh $TAG
for c in wan13b_480p wan14b_720p_w333 hunyuan_720p; do
  timeout -s KILL 200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_${c}_$TAG.json 2> /dev/null
done
timeout -s KILL 200 python tools/bench_passthrough.py > gpurun_out/bench_pt_$TAG.json 2> gpurun_out/bench_pt_$TAG.err
timeout -s KILL 300 python tools/sweep.py --csv gpurun_out/sweep_c4_$TAG.csv > gpurun_out/sweep_$TAG.json 2> gpurun_out/sweep_$TAG.err
timeout -s KILL 120 python tools/trace_attn.py c2 > gpurun_out/trace_$TAG.txt 2>&1
python tools/ncu_summary.py gpurun_out/attn_$TAG.ncu-rep --json gpurun_out/attn_ncu_$TAG.json > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/quant_$TAG.ncu-rep --json gpurun_out/quant_ncu_$TAG.json > /dev/null 2>&1
ncu -i gpurun_out/attn_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/attn_src_$TAG.csv 2>/dev/null
python tools/sass_stalls.py gpurun_out/attn_src_$TAG.csv --top 40 > gpurun_out/attn_stalls_$TAG.txt 2>&1
