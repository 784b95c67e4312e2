# packed cut-element product variants (config 5 probe, 30 steps): built here, run on the box
mkdir -p gpurun_out
T=${1:-cs}
for v in g8 g8m1 pf2 pf2m1 g8m10 g4m6; do
  SC_LIB=paper_2310_14712_b200/libsc_$v.so timeout 600 python scripts/probe_config.py 5 30 > gpurun_out/${T}_$v.log 2>&1
done
