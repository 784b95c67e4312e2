# timing experiment (diagnostics): config-5 step with the explicit update forked against the
# c part (SC_PIPELINE=1) under resource caps, vs the sequential default
mkdir -p gpurun_out
for v in "SC_PIPELINE=0" "SC_PIPELINE=1" "SC_PIPELINE=1 SC_FAR_CAP=1 SC_SOLVE_CTAS_PER_SM=2" "SC_PIPELINE=1 SC_FAR_CAP=1 SC_SOLVE_CTAS_PER_SM=3" "SC_PIPELINE=1 SC_FAR_CAP=1 SC_SOLVE_CTAS_PER_SM=4"; do
  echo "== $v" >> gpurun_out/pipe.log
  env $v python scripts/probe_config.py ${1:-5} 20 2>&1 | python -c "import sys,json; [print(round(json.loads(l)['ms_per_step'],4), json.loads(l)['breakdown_ms']) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/pipe.log
done
