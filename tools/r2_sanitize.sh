# round 2: compute-sanitizer memcheck / racecheck / synccheck / initcheck over the GEMM
# variants (CTA group 1 / 2 / 4), fused and separate CRT, both sizes; summaries -> gpurun_out
mkdir -p gpurun_out
out=gpurun_out/r2_sanitize.log
: > $out
run() {   # tool, timeout, case args...
    tool=$1; to=$2; shift 2
    echo "=== $tool $*" >> $out
    timeout $to compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
        python tools/sanitize_case.py "$@" > /tmp/san.txt 2>&1
    echo "rc=$?" >> $out
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|case m=|Invalid|Race|Barrier|error|hazard" /tmp/san.txt | head -30 >> $out
}
for tool in memcheck synccheck; do
  for cg in 1 2 4; do
    run $tool 900 64 64 64 14 $cg 0
    run $tool 1800 1000 1100 8192 13 $cg 1
    run $tool 1800 1000 1100 8192 13 $cg 0
  done
  run $tool 900 1000 1100 8192 15 2 1 int8
  run $tool 900 300 260 500 13 2 0 fp8 fast
done
run initcheck 1800 1000 1100 8192 13 2 1
run initcheck 900 64 64 64 14 2 0
for cg in 1 2; do
  run racecheck 2400 64 64 64 14 $cg 0
  run racecheck 2400 520 600 8192 13 $cg 1
done
echo done >> $out
