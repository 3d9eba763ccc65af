# kernel-time check: gpu tests + bench (device value only) on the given configs
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in ${CONFIGS:-c2}; do python bench.py --config $c --steps 5 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'ms/solve %.3f kernel %.3f frac %.3f value %.3e'%(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['value']))"; done
