# ncu --set full of the config-5 step kernels (after a plain run of the same command)
mkdir -p gpurun_out
CMD="python scripts/probe_config.py 5 4"
TAG=${1:-prof_c5b}
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k "regex:${2:-k_explicit_3d|k_solve}" -s 4 -c 4 \
  -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
