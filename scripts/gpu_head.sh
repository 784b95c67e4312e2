# HEAD verification: smoke, GPU suite, config-5/4 probes with per-kernel breakdown, config-5 bench line
mkdir -p gpurun_out
T=${1:-h}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu_tests.log
for c in 5 4 2; do timeout 600 python scripts/probe_config.py $c 50 > gpurun_out/${T}_probe_c$c.log 2>&1; done
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_c5.log
