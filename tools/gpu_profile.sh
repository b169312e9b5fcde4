#!/bin/bash
# One GPU session: tests, bench at the driver's command line, launch list and
# ncu --set full captures of the top kernels. Usage: [KERNELS="k_a k_b"] tools/gpu_profile.sh TAG [tests]
TAG=${1:-x}; O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
if [ "$2" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
fi
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> $O/${TAG}_bench.log
GB_PHASES=1 timeout 300 python tools/profile_run.py --iters 4 > $O/${TAG}_phases.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
  python tools/profile_run.py --iters 2 > $O/${TAG}_launches.log 2>&1
for K in ${KERNELS:-k_hvp_rc k_lin_seg k_chi2_tiles}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
    -o $O/${TAG}_$K python tools/profile_run.py --iters 2 > $O/${TAG}_$K.log 2>&1
done
echo done
