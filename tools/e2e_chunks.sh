for i in 1 2; do
echo "== C2"; python tools/e2e_trace.py | tail -2
echo "== C2 prio"; GD_SB_PRIORITY=1 python tools/e2e_trace.py | tail -2
done
GD_TRACE_EXECUTOR=1 python tools/e2e_trace.py 2>&1 | grep -E "unpack|drained|done|e2e" | tail -6
