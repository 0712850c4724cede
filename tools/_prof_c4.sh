# usage: bash tools/_prof_c4.sh LIBTAG CONFIG
FBF_LIB=dl/$1.so python tools/profile_run.py --config $2 > /dev/null 2>&1 && \
FBF_LIB=dl/$1.so ncu --set full --import-source on --clock-control none -k regex:fbf_fused -s 1 -c 1 -o gpurun_out/prof_$2_$1 -f \
  python tools/profile_run.py --config $2 > gpurun_out/ncu_$2_$1.log 2>&1; echo ncu_rc=$?
