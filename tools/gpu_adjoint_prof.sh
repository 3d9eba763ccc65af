# full-scale gradient measurement + ncu captures of the recording persistent
# kernel and the adjoint kernel (C2 scale), launch list
mkdir -p gpurun_out
python tools/adjoint_bench.py > gpurun_out/adjoint_bench.json 2> gpurun_out/adjoint_bench.err
cat gpurun_out/adjoint_bench.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bode_adjoint_kernel -c 1 \
  -o gpurun_out/full_adjoint -f python tools/adjoint_bench.py --reps 1 > gpurun_out/ncu_adjoint.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bode_persistent_kernel -s 1 -c 1 \
  -o gpurun_out/full_recording -f python tools/adjoint_bench.py --reps 1 > gpurun_out/ncu_rec.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_adjoint.csv python tools/adjoint_bench.py --reps 1 > /dev/null 2>&1
tail -n 1 gpurun_out/ncu_adjoint.log; tail -n 1 gpurun_out/ncu_rec.log
