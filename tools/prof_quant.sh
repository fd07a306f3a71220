#!/bin/bash
# ncu capture of the fused quantiser at C2 (40 heads): full set + source counters; summaries in gpurun_out/
mkdir -p gpurun_out
H=${H:-40} timeout 600 ncu --set full --import-source on --clock-control none -k regex:quant_fused -c 1 -s 3 \
  -o gpurun_out/quant_full -f python tools/bench_quant.py > gpurun_out/prof_quant.log 2>&1
ncu -i gpurun_out/quant_full.ncu-rep --page raw --csv > gpurun_out/quant_raw.csv 2>/dev/null
ncu -i gpurun_out/quant_full.ncu-rep --page source --csv > gpurun_out/quant_source.csv 2>/dev/null
ncu -i gpurun_out/quant_full.ncu-rep --page details --csv > gpurun_out/quant_details.csv 2>/dev/null
