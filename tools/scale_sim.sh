# per-rank costs of the N>1 path measured one logical rank at a time on one GPU
# (bench.py --sim-world N --sim-rank r): usage bash tools/scale_sim.sh CONFIG TAG
cfg=${1:-5}; tag=${2:-sim}
for N in 2 4 8; do
  for ((r=0; r<N; r++)); do
    timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --sim-world $N --sim-rank $r \
      > gpurun_out/${tag}_cfg${cfg}_N${N}_r${r}.json 2> /dev/null
  done
done
