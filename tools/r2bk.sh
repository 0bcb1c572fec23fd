# round 2 session 4: compute-sanitizer over the session-4 kernels: k_cast (all storage orders,
# odd / even k, FP8 / INT8 / fast mode), k_digits, the 256x512-tile residue GEMM
mkdir -p gpurun_out
out=gpurun_out/r2bk_sanitize.log
: > $out
run() {   # tool, timeout, case args...
    tool=$1; to=$2; shift 2
    echo "=== $tool $*" >> $out
    start=$(date +%s)
    timeout $to /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
        python tools/sanitize_case.py "$@" > /tmp/san.txt 2>&1
    echo "rc=$? seconds=$(( $(date +%s) - start ))" >> $out
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|case m=|Invalid|Race|Barrier|hazard|last CUDA" /tmp/san.txt | head -20 >> $out; grep -q "ERROR SUMMARY" /tmp/san.txt || head -15 /tmp/san.txt >> $out
}
for t in "N N" "T N" "N T" "T T"; do
  run memcheck 900 300 260 701 13 2 0 fp8 accurate $t 256
done
run memcheck 900 300 260 2300 13 2 0 fp8 accurate T T 256
run memcheck 900 300 260 701 15 2 0 int8 accurate T N 256
run memcheck 900 300 260 701 13 2 0 fp8 fast N T 256
run memcheck 1200 520 600 8192 13 2 1 fp8 accurate N N 512
run memcheck 1200 520 700 16500 13 2 1 fp8 accurate T N 512
run initcheck 900 300 260 701 13 2 0 fp8 accurate T T 256
run synccheck 1200 520 600 8192 13 2 1 fp8 accurate N N 512
echo done >> $out
