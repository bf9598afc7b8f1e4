# SM -> die map probe (research)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/die_probe scripts/die_probe.cu && /tmp/die_probe > gpurun_out/die_probe.txt 2>&1; wc -l gpurun_out/die_probe.txt
