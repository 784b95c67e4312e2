# one round of GPU evidence: tests, bench lines, ncu launch list + full capture (profiles/)
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
timeout 600 python bench.py --config 4 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 600 python bench.py --config 2 --no-cpu > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_launch.log 2>&1 ; echo "rc=$?" >> gpurun_out/ncu_launch.log
timeout 1800 ncu --set full --clock-control none --import-source on -k "regex:k_solve|k_explicit_3d|k_celem" -s 6 -c 6 -o gpurun_out/prof_c5 $CMD > gpurun_out/ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full.log
