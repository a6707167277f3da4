mkdir -p gpurun_out
for rep in 1 2; do
for c in replica tum euroc; do
  (cd ab/r01 && timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' | tail -1 | sed "s/^/r01 $c /") >> gpurun_out/cmp.log
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' | tail -1 | sed "s/^/now $c /" >> gpurun_out/cmp.log
done
done
