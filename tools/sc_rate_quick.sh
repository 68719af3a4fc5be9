timeout 600 python -m pytest tests/test_gpu_sc.py -x -q 2>&1 | tail -2
python tools/sc_rate.py 2>&1 | tail -5
