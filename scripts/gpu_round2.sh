# round evidence (prefix $1): smoke, GPU suite, bench lines, ncu launch list + --set full capture
mkdir -p gpurun_out
T=${1:-r}
nvidia-smi > gpurun_out/${T}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu_tests.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_c5.log
timeout 600 python bench.py --config 4 --no-cpu > gpurun_out/${T}_bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_c4.log
timeout 600 python bench.py --config 2 --no-cpu > gpurun_out/${T}_bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_c2.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_ref.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_c5.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1 ; echo "rc=$?" >> gpurun_out/${T}_ncu_launch.log
timeout 1800 ncu --set full --clock-control none --import-source on -k "regex:k_solve|k_exp3|k_explicit_3d|k_celem" -s 8 -c 8 -o gpurun_out/${T}_prof_c5 $CMD > gpurun_out/${T}_ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_ncu_full.log
