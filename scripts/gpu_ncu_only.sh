# ncu launch list + --set full capture of the config-5 step kernels (after a plain run exits 0)
mkdir -p gpurun_out
T=${1:-n}
CMD="python bench.py --steps 3 --warmup 3 --no-cpu"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_c5.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1 ; echo "rc=$?" >> gpurun_out/${T}_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_solve|k_exp3|k_explicit_3d|k_celem" -s 8 -c 8 -o gpurun_out/${T}_prof_c5 $CMD > gpurun_out/${T}_ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_ncu_full.log
