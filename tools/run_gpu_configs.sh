# one GPU cycle: bench on the replica and stress configs (parity cases elsewhere) -> gpurun_out/
mkdir -p gpurun_out
for c in replica stress; do
timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-replica > gpurun_out/bench_$c.log 2>&1; echo "bench $c exit $?" >> gpurun_out/bench_$c.log
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/bench_stress.log
