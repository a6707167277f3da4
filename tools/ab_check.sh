# correctness of every A/B variant first (the parity tests that exercise the raster paths), then the A/B timing
mkdir -p gpurun_out
for v in $VARIANTS; do
  GS_LIB_PATH=ab/libgs_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_edge.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "${CHECK_K:-backward or forward or chunked}" > gpurun_out/ab_check_$v.log 2>&1
  echo "$v pytest exit $?" >> gpurun_out/ab.log
done
bash tools/ab_quick.sh
