# Configuration matrix through bench.py (one line per configuration) and the
# EuRoC VI bench: tools/run_matrix.sh TAG  (run under gpurun)
TAG=${1:-matrix}
set -x
for a in "--precision fp32" "--precision fp32-bf16" "--mode auto" "--mode dynamic" "--solver schur" "--workload dubrovnik" "--workload dubrovnik --precision fp32" "--workload venice --precision fp32-bf16 --mode dynamic" "--workload venice --precision fp32 --mode dynamic"; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | tail -1 >> gpurun_out/${TAG}_matrix.jsonl
done
timeout 300 python tools/bench_vi.py 2>/dev/null | tail -1 > gpurun_out/${TAG}_vi.jsonl
