# timing experiment: far-d/c-part overlap under resource caps (diagnostics)
mkdir -p gpurun_out
for v in "SC_FAR_CAP=1 SC_SOLVE_CTAS_PER_SM=3" "SC_FAR_CAP=1 SC_SOLVE_CTAS_PER_SM=4" "SC_FAR_CAP=0 SC_SOLVE_CTAS_PER_SM=5" "SC_FAR_CAP=1 SC_SOLVE_CTAS_PER_SM=3 SC_DEBUG_NO_FAR=1"; do
  echo "== $v" >> gpurun_out/ovl2.log
  env $v python scripts/probe_config.py ${1:-4} 200 2>&1 | python -c "import sys,json; [print(round(json.loads(l)['ms_per_step'],4), json.loads(l)['breakdown_ms']) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/ovl2.log
done
