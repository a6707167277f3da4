# A/B: bench value of the in-tree build vs ab/libgs_<v>.so variants, interleaved ($REPS rounds)
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do
for v in base $VARIANTS; do
  if [ $v = base ]; then unset GS_LIB_PATH; else export GS_LIB_PATH=ab/libgs_$v.so; fi
  r=$(timeout 300 python bench.py ${CFG:+--config $CFG} --steps ${STEPS:-40} --warmup 5 --no-cpu-baseline --no-replica 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['value'],1), d['stage_ms_per_step'])")
  echo "$v $r" >> gpurun_out/ab.log
done
done
unset GS_LIB_PATH
