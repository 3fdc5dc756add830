for f in 0.2 0.25 0.3; do for r in 16500 18000; do
python tools/serve_trace.py --rate $r --selection pass --policy none --pass-frac $f --margin-ms 0 2>&1 | grep -E "selection|^rate"
done; done > gpurun_out/serve_trace.txt
