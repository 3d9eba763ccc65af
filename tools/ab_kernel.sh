# A/B timing of the persistent kernel: bench kernel_ms for each config, for
# the in-tree libbode.so and any extra libraries given as BODE_LIBS="a.so b.so"
for lib in "" $BODE_LIBS; do
  for c in ${CONFIGS:-c2 c5 c3}; do
    BODE_LIB=$lib python bench.py --config $c --no-e2e --no-cpu --steps ${STEPS:-10} > gpurun_out/ab.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(sys.argv[1] or 'tree', sys.argv[2], 'kernel_ms %.4f' % d['roofline']['kernel_ms'], 'ms_per_step %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'steps', d['config']['attempted_per_step'])" "$lib" $c
  done
done
