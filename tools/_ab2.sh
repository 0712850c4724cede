set -u
for c in c4 c1 c3 c2 c0; do
  for rep in 1 2; do
    FBF_LIB=dl/base.so timeout 300 python tools/kbench.py --config $c --iters 20 --tag base
    FBF_LIB=dl/nb.so timeout 300 python tools/kbench.py --config $c --iters 20 --tag nb
    FBF_ORDER=rr FBF_LIB=dl/nb.so timeout 300 python tools/kbench.py --config $c --iters 20 --tag nb_rr
  done
done
for o in contig rr; do
FBF_ORDER=$o FBF_LIB=dl/nb.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:fbf_fused -s 1 -c 1 python tools/profile_run.py --config c4 2>&1 | grep -E "dram|duration|hit_rate"
done
