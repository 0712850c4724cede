export FBF_LIB=dl/phases.so FBF_PROF=1
echo "== c1 (pair mode, 7 pairs)"; FBF_MODE=0 timeout 90 python tools/phase_report.py --config c1
echo "== c4 (half mode, warpgroup split)"; FBF_MODE=2 timeout 120 python tools/phase_report.py --config c4 --iters 2
echo "== c3 frame (split mode, 9 pairs)"; FBF_MODE=1 timeout 90 python tools/phase_report.py --config c3
echo "== c2 (duo, split mode)"; FBF_MODE=1 timeout 90 python tools/phase_report.py --config c2 --iters 2
