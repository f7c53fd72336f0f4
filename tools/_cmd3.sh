timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "hubs or config3 or hand or spec or random_small or delta_le or ppsp" 2>&1 | tail -2
for CL in 4 16; do
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DGI_CLAIMS=$CL -lineinfo -Xcompiler -fPIC -shared -I include -o paper_1911_07260_b200/libgi.so paper_1911_07260_b200/csrc/gi_kernels.cu paper_1911_07260_b200/csrc/gi_capi.cu
for d in 1 2 8; do echo -n "CL=$CL cfg3 d$d: "; timeout 100 python bench.py --config 3 --delta $d --steps 5 --warmup 3 --no-cpu-baseline --no-compare 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); c=j['counters']; print(round(j['ms_per_step'],3), c['rounds'], c['spills'], c['vertices_processed'])"; done
echo -n "CL=$CL cfg3 d2 pre_read off: "; timeout 100 python bench.py --config 3 --delta 2 --pre-read 2 --steps 5 --warmup 3 --no-cpu-baseline --no-compare 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); c=j['counters']; print(round(j['ms_per_step'],3), c['rounds'], c['spills'], c['vertices_processed'])"
done
