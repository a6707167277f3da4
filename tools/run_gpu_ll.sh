# launch list (ncu gpu__time_duration) of one bench step of config $1 -> gpurun_out/launches_$1.csv
mkdir -p gpurun_out
timeout 600 python bench.py --config $1 --launch-list > gpurun_out/ll_$1.log 2>&1 && timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python bench.py --config $1 --launch-list > gpurun_out/ncu_ll_$1.log 2>&1; echo "exit $?" >> gpurun_out/ncu_ll_$1.log
