# setup-time breakdown on config 5 + the parity tests that exercise the cut-cell matrices
mkdir -p gpurun_out
T=${1:-s}
SC_SETUP_TIMES=1 timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/${T}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_celldt.py -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
