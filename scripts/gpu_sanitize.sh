mkdir -p gpurun_out
for T in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 50 --log-file gpurun_out/r2_sanitize_$T.log python scripts/sanitize_run.py > gpurun_out/r2_sanitize_$T.out 2>&1
  echo "$T rc=$?"; tail -3 gpurun_out/r2_sanitize_$T.log
done
