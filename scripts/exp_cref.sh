# reference-element product tile variants (CR_EPW elements per warp x CR_NW warps; config 5 and 4
# probes), then the round evidence with the default library
mkdir -p gpurun_out
T=${1:-cr}
for v in r48 r86 r82 r68; do
  SC_LIB=paper_2310_14712_b200/libsc_$v.so timeout 400 python scripts/probe_config.py 5 30 > gpurun_out/${T}_c5_$v.log 2>&1
done
timeout 400 python scripts/probe_config.py 5 30 > gpurun_out/${T}_c5_default.log 2>&1
for v in r48 r86; do
  SC_LIB=paper_2310_14712_b200/libsc_$v.so timeout 300 python scripts/probe_config.py 4 50 > gpurun_out/${T}_c4_$v.log 2>&1
done
timeout 300 python scripts/probe_config.py 4 50 > gpurun_out/${T}_c4_default.log 2>&1
bash scripts/gpu_round2.sh $T
