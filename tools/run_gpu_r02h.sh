# round-2 evidence after the quadrant-group backward: GPU tests, smoke, bench lines of every
# config, reference arm, launch lists, ncu --set full of the backward kernels -> gpurun_out/
bash tools/run_gpu_r02_final.sh
CFG=replica bash tools/run_ncu.sh "k_raster_bwdq" 3
