# A/B of programmatic dependent launch: bench with and without, alternating
mkdir -p gpurun_out
for k in 1 2; do
  GS_PDL=1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/pdl1_$k.log 2>&1
  GS_PDL=0 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/pdl0_$k.log 2>&1
done
