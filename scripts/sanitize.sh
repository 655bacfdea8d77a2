# compute-sanitizer memcheck over every kernel variant (small inputs), one tool per call.
mkdir -p gpurun_out
TOOL=${TOOL:-memcheck}
for k in auto tma general pipe; do
  U16M_TEST_SMALL=1 U16M_KERNEL=$k timeout 900 compute-sanitizer --tool $TOOL --error-exitcode 9 \
     python tests/gpu_helpers/variant_check.py > gpurun_out/sanitize_${TOOL}_$k.log 2>&1
  echo "$TOOL $k rc=$?"; tail -3 gpurun_out/sanitize_${TOOL}_$k.log
done
