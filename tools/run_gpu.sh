# one GPU cycle: parity tests, bench, per-launch list (ncu) [, full ncu capture of $NCU_K]
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 300 python bench.py --launch-list > gpurun_out/ll_plain.log 2>&1 && timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --launch-list > gpurun_out/ncu_ll.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_ll.log
if [ -n "$NCU_K" ]; then
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"$NCU_K" -c ${NCU_C:-6} -o gpurun_out/prof python bench.py --launch-list > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?" >> gpurun_out/ncu_full.log
fi
