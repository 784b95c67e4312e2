# ncu --set full of the candidate explicit kernel in the harness (diagnostics)
mkdir -p gpurun_out
T=${1:-hn}; B=${2:-scripts/exp_harness}; RX=${3:-k_exp3}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${RX}" -s 1 -c 1 -o gpurun_out/$T $B 160 1 0 > gpurun_out/${T}_ncu.log 2>&1
echo rc=$? >> gpurun_out/${T}_ncu.log
