# adjoint (gradient) path: GPU tests, forward bench regression check
python -m pytest tests/test_gpu_adjoint.py -x -q 2>&1 | tail -30
python bench.py --config c2 --steps 10 --no-cpu --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2', d['ms_per_step'], d['roofline']['kernel_ms'])"
