echo "== C2"; python tools/e2e_trace.py | tail -2
echo "== C4"; python tools/e2e_trace.py --ligands 1000 --atoms 120 --rotamers 32 | tail -2
echo "== C5"; python tools/e2e_trace.py --dims 47 --spacing 0.375 | tail -2
GD_TRACE_EXECUTOR=1 python tools/e2e_trace.py 2>&1 | tail -12
GD_TRACE_EXECUTOR=1 python tools/e2e_trace.py --ligands 1000 --atoms 120 --rotamers 32 2>&1 | tail -12
