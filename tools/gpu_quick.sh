# quick GPU check: gpu tests + e2e probe + c2 bench
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/e2e_probe.py
python bench.py --config c2 --steps 5 --no-cpu
