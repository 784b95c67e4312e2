# GPU suite + config-5 bench line (evidence after a kernel change)
mkdir -p gpurun_out
T=${1:-q}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu_tests.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_c5.log
