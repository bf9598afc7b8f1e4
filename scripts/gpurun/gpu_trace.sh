mkdir -p gpurun_out
python scripts/trace_step.py --h 5120 --heads 40 --mesh 4x2 --chunks 1,4 > gpurun_out/trace_cfg4_42.jsonl 2>&1
python scripts/trace_step.py --h 4096 --heads 32 --mesh 4x2 --chunks 1,2,4 > gpurun_out/trace_cfg3_42.jsonl 2>&1
python scripts/trace_step.py --h 4096 --heads 32 --mesh 1x1 --chunks 1 > gpurun_out/trace_n1.jsonl 2>&1
python scripts/trace_step.py --h 4096 --heads 32 --mesh 4x2 --chunks 4 --ops > gpurun_out/trace_cfg3_42_c4_ops.txt 2>&1
cat gpurun_out/trace_cfg4_42.jsonl gpurun_out/trace_cfg3_42.jsonl gpurun_out/trace_n1.jsonl
