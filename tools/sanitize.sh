# compute-sanitizer over every kernel family (tools/sanitize_run.py); logs in gpurun_out/
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for part in ${PARTS:-analytic mlp program adjoint mlp_adjoint}; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py $part \
      > gpurun_out/sanitize_${tool}_${part}.log 2>&1
    echo "$tool $part rc=$?" >> gpurun_out/sanitize_summary.txt
  done
done
cat gpurun_out/sanitize_summary.txt
