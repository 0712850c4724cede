# dev: device-resident timing of every dl/*.so on the given configs. Usage: bash tools/exp.sh c1 [c3 ...]
for c in "$@"; do
  for lib in dl/*.so; do FBF_LIB=$lib timeout 120 python tools/kbench.py --config $c --iters 40 --tag "$(basename $lib .so)"; done
done
