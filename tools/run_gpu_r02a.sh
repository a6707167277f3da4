# round-2 first cycle: parity tests, smoke, bench on tum and replica
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_tum.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_tum.log
timeout 400 python bench.py --config replica --steps 20 --warmup 5 --no-cpu-baseline --no-replica > gpurun_out/bench_replica.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_replica.log
