# MLP adjoint evidence (C4 scale): timing JSON, launch list, and one
# --set full capture each of a VJP launch (stage 3) and a weight-gradient launch
mkdir -p gpurun_out
python tools/adjoint_bench.py --config c4 --reps 5 > gpurun_out/adjoint_bench_c4.json 2> gpurun_out/adjoint_bench_c4.err
cat gpurun_out/adjoint_bench_c4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_mlp_adjoint.csv python tools/adjoint_bench.py --config c4 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"vjp_kernel|wg_kernel" -s 4 -c 2 \
  -o gpurun_out/full_mlp_adjoint_tc -f python tools/adjoint_bench.py --config c4 --reps 1 > gpurun_out/ncu_full_mlp_adjoint.log 2>&1
tail -2 gpurun_out/ncu_full_mlp_adjoint.log
