# correctness (ragged, masked) + config-5-size timing of selected harness builds (diagnostics)
mkdir -p gpurun_out
T=$1; shift
{ for b in "$@"; do echo "=== $b"; timeout 120 $b 160 10 0 | grep -E "cand|regs|flag 1"; timeout 60 $b 37 3 1 41 29 | grep -E "cand vs|differing"; timeout 60 $b 13 3 0 19 14 | grep -E "cand vs|differing"; done; } > gpurun_out/${T}.log 2>&1
