# compute-sanitizer tiers on small inputs -> gpurun_out/sanitizer_*.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for args in "tiny 0" "tum 2 20000" "tum 0 20000" "euroc 2 20000 3"; do
    tag=$(echo "$tool $args" | tr ' ' '_')
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_step.py $args > gpurun_out/sanitizer_$tag.log 2>&1
    echo "exit $?" >> gpurun_out/sanitizer_$tag.log
  done
done
grep -H "ERROR SUMMARY\|^exit" gpurun_out/sanitizer_*.log > gpurun_out/sanitizer_summary.txt
