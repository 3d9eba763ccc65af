python tools/adjoint_bench.py --reps 3
timeout 900 ncu --set full --clock-control none -k regex:bode_persistent_kernel -s 1 -c 1 -o gpurun_out/full_recording -f python tools/adjoint_bench.py --reps 1 > gpurun_out/ncu_rec.log 2>&1; tail -1 gpurun_out/ncu_rec.log
