# ncu --set full (with source) of ONE sub-kernel of a config's step, after a plain run of
# the same command.  usage: bash scripts/ncu_kernel.sh TAG CONFIG WHICH KERNEL_REGEX
mkdir -p gpurun_out
TAG=$1; CFG=$2; WHICH=$3; RX=$4
CMD="python scripts/prof_kernel.py $CFG $WHICH 3"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed" >> gpurun_out/${TAG}_plain.log; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:${RX}" -s 1 -c 1 \
  -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
