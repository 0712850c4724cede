# usage: bash tools/_prof1.sh CONFIG TAG  -- one ncu --set full capture of the fused kernel
python tools/profile_run.py --config $1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fbf_fused -s 1 -c 1 -o gpurun_out/prof_$1_$2 -f \
  python tools/profile_run.py --config $1 > gpurun_out/ncu_$1_$2.log 2>&1; echo ncu_rc=$?
