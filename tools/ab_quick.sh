# A/B with bench.py --quick: in-tree build vs ab/libgs_<v>.so variants, interleaved ($REPS rounds)
mkdir -p gpurun_out
for rep in $(seq ${REPS:-3}); do
for c in ${CONFIGS:-replica}; do
for v in base $VARIANTS; do
  if [ $v = base ]; then unset GS_LIB_PATH; else export GS_LIB_PATH=ab/libgs_$v.so; fi
  r=$(timeout 300 python bench.py --config $c --quick --steps ${STEPS:-100} --warmup 5 2>/dev/null | tail -1)
  echo "$c $v $r" >> gpurun_out/ab.log
done
done
done
unset GS_LIB_PATH
