mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mlp_fused -c 1 -o gpurun_out/c4_fused -f python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_c4.log 2>&1
tail -5 gpurun_out/ncu_c4.log
