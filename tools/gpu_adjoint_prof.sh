# full-scale gradient measurement + ncu capture of the adjoint kernel
mkdir -p gpurun_out
python tools/adjoint_bench.py > gpurun_out/adjoint_bench.json 2> gpurun_out/adjoint_bench.err
cat gpurun_out/adjoint_bench.json; tail -3 gpurun_out/adjoint_bench.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bode_adjoint_kernel -c 1 \
  -o gpurun_out/full_adjoint -f python tools/adjoint_bench.py --reps 1 > gpurun_out/ncu_adjoint.log 2>&1
tail -2 gpurun_out/ncu_adjoint.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_adjoint.csv python tools/adjoint_bench.py --reps 1 > /dev/null 2>&1
