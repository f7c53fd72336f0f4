REBUILD=1 timeout 900 python tools/trace_async.py cfg4 2 bsp 2>&1 | grep -v "^CTA0  [0-4] "
