timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "not slow and not config4" 2>&1 | tail -2
for d in 1 2 4 8; do echo -n "cfg3 d$d: "; timeout 100 python bench.py --config 3 --delta $d --steps 5 --warmup 3 --no-cpu-baseline --no-compare 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); c=j['counters']; print(round(j['ms_per_step'],3), c['rounds'], c['spills'])"; done
echo -n "cfg2: "; timeout 100 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-compare 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['ms_per_step'],3))"
echo -n "cfg1: "; timeout 100 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline --no-compare 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['ms_per_step'],3))"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DGI_TRACE -Xcompiler -fPIC -shared -I include -o /tmp/libgi_trace.so paper_1911_07260_b200/csrc/gi_kernels.cu paper_1911_07260_b200/csrc/gi_capi.cu
for a in "cfg3 1 bsp" "cfg3 8 bsp"; do timeout 120 python tools/trace_async.py $a 2>&1 | grep -v CTA0; done
