python -m pytest tests/test_gpu_parity.py tests/test_gpu_solver.py tests/test_gpu_adjoint.py -q -x 2>&1 | tail -3
for c in c2 c5 c3; do python bench.py --config $c --steps 10 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), d['roofline']['frac'])"; done
