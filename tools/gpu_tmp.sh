timeout -s KILL 60 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2i.txt 2>&1; echo "EXIT $?" >> gpurun_out/smoke_r2i.txt
timeout -s KILL 400 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 120 > gpurun_out/tests_r2i.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_r2i.txt
timeout -s KILL 180 python tools/bench_passthrough.py > gpurun_out/bench_pt_r2i.json 2> gpurun_out/bench_pt_r2i.err
timeout -s KILL 300 python tools/sweep.py --fidelity --csv gpurun_out/sweep_c4_fid_r2i.csv > gpurun_out/sweep_fid_r2i.json 2> gpurun_out/sweep_fid_r2i.err
