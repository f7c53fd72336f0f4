# usage: bash tools/sweep_cfg.sh  -> gpurun_out/cfg*_*.json
for d in 8192 32768; do timeout 200 python bench.py --config 2 --delta $d --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/cfg2_d$d.json 2>gpurun_out/cfg2_d$d.err; done
for d in 1 2 4 8; do timeout 300 python bench.py --config 3 --delta $d --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/cfg3_d$d.json 2>gpurun_out/cfg3_d$d.err; done
timeout 200 python bench.py --config 1 --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/cfg1.json 2>gpurun_out/cfg1.err
for gc in 8 16 37; do timeout 600 python bench.py --config 5 --delta 32768 --group-ctas $gc --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/cfg5_g$gc.json 2>gpurun_out/cfg5_g$gc.err; done
