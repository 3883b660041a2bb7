# every workload's bench line (product defaults) into gpurun_out/${TAG}_bench_<workload>.json
TAG=${1:-r}
for w in weak single deflation tiny arnoldi; do
  timeout 900 python bench.py --workload $w ${BENCH_ARGS:---steps 10 --warmup 3} > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
done
