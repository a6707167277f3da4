# full ncu capture of kernels matching $1 (first ${2:-6} launches) of one tum bench step -> gpurun_out/prof.ncu-rep
mkdir -p gpurun_out
timeout 300 python bench.py --launch-list ${CFG:+--config $CFG} > gpurun_out/ll_plain.log 2>&1 && timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"$1" --launch-skip ${SKIP:-0} -c ${2:-6} -o gpurun_out/prof python bench.py --launch-list ${CFG:+--config $CFG} > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?" >> gpurun_out/ncu_full.log
