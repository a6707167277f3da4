# one GPU cycle: parity tests + bench on tum (headline) and the multi-view configs -> gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
for c in ${CONFIGS:-euroc stress}; do
timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-replica > gpurun_out/bench_$c.log 2>&1; echo "bench $c exit $?" >> gpurun_out/bench_$c.log
done
