#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small solver runs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_san.log 2>&1 || { echo build failed; exit 1; }
OUT=gpurun_out/sanitize.log; : > $OUT
for tool in memcheck racecheck synccheck; do
  for case in whole split concurrent retry strip crr tree; do
    if [ $tool != memcheck ] && { [ $case = crr ] || [ $case = tree ]; }; then continue; fi
    echo "=== $tool $case" >> $OUT
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 17 python scripts/sanitize_case.py $case >> $OUT 2>&1
    echo "rc=$?" >> $OUT
  done
done
grep -E "^===|^rc=|ERROR SUMMARY|RACECHECK SUMMARY|hazard" $OUT | head -80
