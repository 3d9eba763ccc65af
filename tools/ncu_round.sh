# ncu evidence for profiles/: launch lists (cold, serialised) and one
# --set full capture of the dominant kernel, per config in $CONFIGS
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c4}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
  case $c in c4) k=mlp_fused_kernel;; *) k=bode_persistent_kernel;; esac
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 \
    -o gpurun_out/full_$c -f python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_$c.log 2>&1
  tail -2 gpurun_out/ncu_full_$c.log
done
ls -la gpurun_out
