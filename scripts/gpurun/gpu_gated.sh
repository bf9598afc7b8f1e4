# Gated / fused / signalled parity, then per-rank compute with and without gating.
timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider -k "gated or fused or signalled" 2>&1 | tail -3
timeout 300 python scripts/emulate_mesh.py --cfg 3,4 --meshes 8x1,4x2 --chunks 1,2,4 > gpurun_out/emu_nogate.jsonl 2> gpurun_out/emu.err
timeout 300 python scripts/emulate_mesh.py --cfg 3,4 --meshes 8x1,4x2 --chunks 2,4 --gated > gpurun_out/emu_gate.jsonl 2>> gpurun_out/emu.err
timeout 300 python bench.py 2>/dev/null | tail -1
