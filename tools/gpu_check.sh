# full GPU check: tests, bench at the driver's command line. usage: tools/_cmd_full.sh TAG
TAG=$1; O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> $O/${TAG}_bench.log
