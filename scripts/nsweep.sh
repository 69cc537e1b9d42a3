for N in 512 1024 2048 4096; do
  timeout 300 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-e2e --n-samples $N > gpurun_out/ns_C3_N${N}_w4.json 2>/dev/null
done
timeout 300 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-e2e --n-samples 2048 --cta-warps 8 > gpurun_out/ns_C3_N2048_w8.json 2>/dev/null
