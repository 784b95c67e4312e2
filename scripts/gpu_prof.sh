# one ncu --set full capture of the top step kernels (run after the plain command exits 0)
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-cpu"
TAG=${1:-prof}
KREGEX=${2:-"k_solve|k_explicit_3d"}
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX}" -s 6 -c 4 \
  -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
