# compute-sanitizer over tools/sanitize_case.py: memcheck,
# racecheck (shared-memory hazards), synccheck (barrier misuse), initcheck.
# usage: bash tools/sanitize.sh <out-prefix>   (logs in gpurun_out/)
P=${1:-r02}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --launch-timeout 0 --error-exitcode 9 \
    --log-file gpurun_out/${P}_sanitize_${tool}.log python tools/sanitize_case.py \
    > gpurun_out/${P}_sanitize_${tool}.out 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/${P}_sanitize_${tool}.out)"
done
