timeout 300 python -m pytest tests/test_gpu_stencil.py -x -q 2>&1 | tail -3
bash scripts/gpu_tma.sh tma1
