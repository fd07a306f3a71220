timeout -s KILL 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r3t.txt 2>&1; echo "EXIT $?" >> gpurun_out/smoke_r3t.txt
timeout -s KILL 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider --timeout 200 > gpurun_out/tests_r3t.txt 2>&1; echo "EXIT $?" >> gpurun_out/tests_r3t.txt
