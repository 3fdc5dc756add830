for f in 0.15; do for r in 19500 20500; do
python tools/serve_trace.py --rate $r --selection pass --policy none --pass-frac $f --margin-ms 0 2>&1 | grep -E "^rate" | sed "s/^/frac $f /"
done; done > gpurun_out/serve_trace.txt
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
