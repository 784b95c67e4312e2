# ND leaf-size experiment (diagnostics): solve time and factor size
mkdir -p gpurun_out
for L in 32 64 128 256; do
  for c in 4 5; do
    echo "== leaf $L config $c" >> gpurun_out/leaf.log
    SC_ND_LEAF=$L python scripts/probe_config.py $c 20 2>&1 | python -c "import sys,json; [print(round(json.loads(l)['ms_per_step'],4), json.loads(l)['breakdown_ms'], json.loads(l)['nnz_factor'], json.loads(l)['n_supernodes'], round(json.loads(l)['setup_s'],1)) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/leaf.log
  done
done
