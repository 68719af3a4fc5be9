timeout 900 python bench.py --steps 50 2>&1 | tail -2
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1
