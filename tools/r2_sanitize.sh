# round 2: compute-sanitizer memcheck / synccheck / racecheck / initcheck over the GEMM
# variants (CTA group 1 / 2 / 4), fused and separate CRT, INT8 and fast mode; summaries ->
# gpurun_out/r2_sanitize.log (each case: rc and the tool's summary lines)
mkdir -p gpurun_out
out=gpurun_out/r2_sanitize.log
: > $out
run() {   # tool, timeout, case args...
    tool=$1; to=$2; shift 2
    echo "=== $tool $*" >> $out
    start=$(date +%s)
    timeout $to compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
        python tools/sanitize_case.py "$@" > /tmp/san.txt 2>&1
    echo "rc=$? seconds=$(( $(date +%s) - start ))" >> $out
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|case m=|Invalid|Race|Barrier|hazard|last CUDA" /tmp/san.txt | head -20 >> $out
}
for cg in 1 2 4; do
  run memcheck 900 64 64 64 14 $cg 0
  run memcheck 1200 520 600 8192 13 $cg 1
done
run memcheck 900 520 600 8192 15 2 1 int8
run memcheck 900 300 260 500 13 2 0 fp8 fast
run memcheck 900 300 260 2300 13 2 0 karatsuba
for cg in 1 2 4; do
  run synccheck 1200 520 600 8192 13 $cg 1
done
run synccheck 900 64 64 64 14 2 0
run initcheck 1200 520 600 8192 13 2 1
for cg in 1 2; do
  run racecheck 1800 64 64 64 14 $cg 0
done
run racecheck 2400 520 600 8192 13 2 1
echo done >> $out
