# config-5-size timing of each harness build (diagnostics)
mkdir -p gpurun_out
T=${1:-hb}
{ for b in scripts/exp_harness_*; do case "$b" in *.cu|*.sh) continue;; esac; echo "=== $b"; timeout 120 $b 160 10 0 | grep -E "cand:|product|regs"; done; } > gpurun_out/${T}.log 2>&1
