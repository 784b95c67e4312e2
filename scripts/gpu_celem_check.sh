# c-element product tests + config-5 timing (after a k_celem change)
mkdir -p gpurun_out
T=${1:-ce}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hrz.py tests/test_gpu_leapfrog.py tests/test_gpu_energy.py tests/test_gpu_stress.py tests/test_gpu_bell.py -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 600 python scripts/probe_config.py 5 20 2>&1 | python -c "import sys,json; [print(round(json.loads(l)['ms_per_step'],4), json.loads(l)['breakdown_ms']) for l in sys.stdin if l.startswith('{')]" > gpurun_out/${T}_probe.log 2>&1
