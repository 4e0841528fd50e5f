python tools/e2e_trace.py
for c0 in 1250 2500; do echo "== first $c0 x4"; GD_CHUNK0=$c0 python tools/e2e_trace.py | tail -1; done
echo "== one chunk"; GD_CHUNK=10000 python tools/e2e_trace.py | tail -1
