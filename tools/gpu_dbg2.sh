for v in plain single; do timeout 120 python tools/debug_graph2.py $v 2>&1 | grep -v "^  File" | tail -6; done
