# timing experiment (diagnostics): config-5 step sequential vs pipelined (SC_PIPELINE=1: far-d
# explicit update of step n+1 forked against the c part of step n), experiment build
mkdir -p gpurun_out
T=${1:-pipe2}
for v in "SC_PIPELINE=0" "SC_PIPELINE=1" "SC_PIPELINE=1 SC_SOLVE_CTAS_PER_SM=4" "SC_PIPELINE=1 SC_FAR_CAP=1"; do
  echo "== $v" >> gpurun_out/${T}.log
  env SC_LIB=$PWD/paper_2310_14712_b200/libsc_exp.so $v timeout 600 python scripts/probe_config.py 5 20 2>&1 | python -c "import sys,json; [print(round(json.loads(l)['ms_per_step'],4), json.loads(l)['breakdown_ms']) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/${T}.log
done
