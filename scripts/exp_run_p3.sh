# p = 3 harness builds at config-4 size (64^3) and 128^3 (diagnostics)
mkdir -p gpurun_out
T=${1:-hp3}
{ for b in scripts/exp_harness_p3_*; do echo "=== $b"; for n in 64 128; do timeout 120 $b $n 20 0 | grep -E "cand:|product|cand vs|flag 1"; done; timeout 60 $b 37 3 1 41 29 | grep -E "cand vs|differing"; done; } > gpurun_out/${T}.log 2>&1
