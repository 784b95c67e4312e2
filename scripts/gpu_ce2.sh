# packed cut-element products: c-path tests + probes + bench line
mkdir -p gpurun_out
T=${1:-ce}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config5.py tests/test_gpu_hrz.py tests/test_gpu_leapfrog.py tests/test_gpu_energy.py tests/test_gpu_stress.py tests/test_gpu_bell.py -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
for c in 5 4; do timeout 600 python scripts/probe_config.py $c 50 > gpurun_out/${T}_probe_c$c.log 2>&1; done
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_c5.log
