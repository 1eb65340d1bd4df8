# compute-sanitizer over scripts/sanitize_cases.py. Writes
# gpurun_out/sanitize_<tool>_<case>.log and a summary line per run.
# The conv case (persistent tcgen05 cta_group::2 kernels) made no progress under
# any of the three tools within 900 s and is left out (QRM_SANITIZE_CONV=1 adds it).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  cases="decode host rs tiles"; [ -n "$QRM_SANITIZE_CONV" ] && cases="$cases conv"
  for c in $cases; do
    timeout ${QRM_SANITIZE_TIMEOUT:-600} compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize_cases.py $c \
      > gpurun_out/sanitize_${tool}_${c}.log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${c}.log | tail -1)"
  done
done | tee gpurun_out/sanitize_summary.txt
