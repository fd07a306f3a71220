bash tools/gpu_dev.sh r1n
