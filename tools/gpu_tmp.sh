for tool in memcheck racecheck synccheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool python tools/sanitize_small.py > gpurun_out/sanitizer_${tool}_r2z.txt 2>&1; echo "EXIT $?" >> gpurun_out/sanitizer_${tool}_r2z.txt
done
