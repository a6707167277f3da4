# euroc (16 views per GPU) bench + launch list
mkdir -p gpurun_out
timeout 300 python bench.py --config euroc --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/euroc.log 2>&1
timeout 300 python bench.py --config euroc --launch-list > gpurun_out/ll_e.log 2>&1 && timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_euroc.csv python bench.py --config euroc --launch-list > gpurun_out/ncu_lle.log 2>&1
