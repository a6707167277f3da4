mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for c in replica tum euroc; do bash tools/run_gpu_ll.sh $c; done
CFG=replica bash tools/run_ncu.sh "k_raster_bwdq" 3
