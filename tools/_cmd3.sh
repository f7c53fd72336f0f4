for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "kcore" 2>&1 | tail -1; done
for c in 2 3; do echo -n "kcore cfg$c: "; timeout 300 python bench.py --config $c --app kcore --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['ms_per_step'],3), j['parity'])"; done
