# GPT layer per-rank trace at cfg 4 (4,2): where chunking costs
mkdir -p gpurun_out
timeout 300 python scripts/trace_step.py --layer gpt --h 5120 --heads 40 --mesh 4x2 --chunks 4,1 --gemm-ctas 132 --ops > gpurun_out/r02_trace_gpt42.txt 2>&1
grep '"mesh"' gpurun_out/r02_trace_gpt42.txt | cut -c1-1500
