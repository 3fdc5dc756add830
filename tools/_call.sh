for f in 0.2 0.25; do for r in 16000 19000 22000; do
python tools/serve_trace.py --rate $r --margin-ms 0 --selection pass --policy none --pass-frac $f 2>&1 | grep -v "^late"
done; done > gpurun_out/serve_trace.txt
