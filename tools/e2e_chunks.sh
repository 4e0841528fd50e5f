for cfg in "625 4" "1250 8" "625 16" "1000 3" "400 6" "2000 8"; do set -- $cfg; echo "== first $1 growth $2"; GD_CHUNK0=$1 GD_CHUNK_GROWTH=$2 python tools/e2e_trace.py | tail -2; done
