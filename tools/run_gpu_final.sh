# one full GPU cycle for the round's evidence: parity tests, smoke, bench lines (tum with the CPU
# baseline, euroc, stress), the reference arm, the per-launch list and ncu --set full of the top kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
for c in euroc stress; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-replica > gpurun_out/bench_$c.log 2>&1; echo "bench $c exit $?" >> gpurun_out/bench_$c.log
done
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
timeout 300 python bench.py --launch-list > gpurun_out/ll_plain.log 2>&1 && timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --launch-list > gpurun_out/ncu_ll.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_ll.log
timeout 300 python bench.py --config euroc --launch-list > gpurun_out/ll_plain_e.log 2>&1 && timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_euroc.csv python bench.py --config euroc --launch-list > gpurun_out/ncu_ll_e.log 2>&1; echo "ncu euroc exit $?" >> gpurun_out/ncu_ll_e.log
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"${NCU_K:-k_raster|k_adam|k_preprocess|k_tile_sort|k_bin|k_ssim}" -c ${NCU_C:-30} -o gpurun_out/prof python bench.py --launch-list > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?" >> gpurun_out/ncu_full.log
