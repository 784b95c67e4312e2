# run the explicit-kernel harness variants on the GPU box (diagnostics)
mkdir -p gpurun_out
T=${1:-h}
{
for b in scripts/exp_harness*; do
  [ -x "$b" ] || continue
  case "$b" in *.cu|*.sh) continue;; esac
  echo "=== $b"
  timeout 120 $b 160 10 0
  timeout 60 $b 37 3 1 41 29
  timeout 60 $b 13 3 0 19 14
done
} > gpurun_out/${T}.log 2>&1
