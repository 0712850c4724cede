FBF_STREAM_BANDS=8 timeout 60 python tools/stream_check.py c1
for nb in 8 16; do FBF_TRACE=1 FBF_STREAM_BANDS=$nb timeout 60 python tools/e2e_probe.py 2>&1 | tail -2; done
