# Round 2: GEMM DRAM traffic vs L2 cache hints / raster group at the h=12288 shapes;
# per-rank emulation with the post-all-reduce elementwise step on the compute stream.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_gpt.py tests/test_gpu_graph.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -3
G="python scripts/gemm_bench.py --h 12288 --no-ref"
for hint in 0 1 8 9 3 5; do
  for gm in rule 4 16; do
    if [ $gm = rule ]; then unset ATP_GROUP_M; else export ATP_GROUP_M=$gm; fi
    export ATP_L2HINT=$hint
    echo "== hint $hint group $gm" >> gpurun_out/r02_l2_sweep.log
    timeout 300 $G --iters 5 >> gpurun_out/r02_l2_sweep.log 2>&1
    timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:gemm_sm100 --launch-skip 3 --launch-count 1 --csv $G --iters 1 --only fc2_fwd > gpurun_out/r02_l2_ncu_h${hint}_g${gm}.csv 2>/dev/null
    timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:gemm_sm100 --launch-skip 3 --launch-count 1 --csv $G --iters 1 --only qkv_fwd > gpurun_out/r02_l2_ncu_qkv_h${hint}_g${gm}.csv 2>/dev/null
  done
done
unset ATP_GROUP_M ATP_L2HINT
grep -c tflops gpurun_out/r02_l2_sweep.log
for ew in 1 0; do
  ATP_EW_COMPUTE=$ew timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1 --chunks 1,2,4 --gemm-ctas 132 >> gpurun_out/r02_emul_ew$ew.jsonl 2>>gpurun_out/r02_emul.err
  ATP_EW_COMPUTE=$ew timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2 --chunks 1,4 --gemm-ctas 148 >> gpurun_out/r02_emul_ew$ew.jsonl 2>>gpurun_out/r02_emul.err
done
cat gpurun_out/r02_emul_ew1.jsonl gpurun_out/r02_emul_ew0.jsonl
timeout 300 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 1,4 --gemm-ctas 132 > gpurun_out/r02_trace_42_ew1_cap132.txt 2>&1
tail -2 gpurun_out/r02_trace_42_ew1_cap132.txt | cut -c1-600
