python -m pytest tests -q -m gpu --tb=short 2>&1 | tail -15
timeout 600 python bench.py --steps 200 --warmup 20 2>&1 | tail -5
