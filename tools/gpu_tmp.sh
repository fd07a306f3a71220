timeout -s KILL 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r3c.txt 2>&1; echo "EXIT $?" >> gpurun_out/smoke_r3c.txt
