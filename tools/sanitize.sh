# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the
# small-shape cases of tools/sanitize_cases.py, one log per tool and case
# under gpurun_out/sanitize/.  Run on the B200 box:
#   gpurun -- 'bash tools/sanitize.sh'
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for case in k1 k2_dense k2_pair band k3_grouped cosine dedup; do
  for tool in memcheck racecheck synccheck initcheck; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check full"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --error-exitcode 99 \
        python tools/sanitize_cases.py $case > gpurun_out/sanitize/${tool}_${case}.log 2>&1
    echo "$tool $case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize/${tool}_${case}.log | tail -1)"
  done
done
