set -x
for a in "--precision fp32" "--precision fp32-bf16" "--mode auto" "--mode dynamic" "--solver schur" "--workload dubrovnik" "--workload dubrovnik --precision fp32" "--workload venice --precision fp32-bf16 --mode dynamic"; do
  timeout 600 python bench.py --steps 5 --warmup 3 $a 2>/dev/null | tail -1 >> gpurun_out/s119_matrix.jsonl
done
timeout 300 python tools/bench_vi.py 2>/dev/null | tail -1 > gpurun_out/s119_vi.jsonl
