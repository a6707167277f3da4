# A/B per-kernel device times: ncu launch list (gpu__time_duration.sum) of one bench step for the
# in-tree build and each ab/libgs_<v>.so in $VARIANTS -> gpurun_out/ll_<v>.csv
mkdir -p gpurun_out
for v in base $VARIANTS; do
  if [ $v = base ]; then unset GS_LIB_PATH; else export GS_LIB_PATH=ab/libgs_$v.so; fi
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ll_$v.csv python bench.py ${CFG:+--config $CFG} --launch-list > gpurun_out/ncu_ll_$v.log 2>&1
  echo "$v exit $?" >> gpurun_out/ncu_ll_$v.log
done
unset GS_LIB_PATH
