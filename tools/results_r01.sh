#!/bin/bash
# Round-1 results: every bench line the DESIGN.md §10 tables quote, one JSON line each,
# into gpurun_out/results.jsonl (copied to profiles/ afterwards). Run on the GPU box.
out=gpurun_out/results.jsonl
: > $out
run() { timeout 900 python bench.py "$@" --no-cpu-baseline 2>/dev/null | tail -1 >> $out; }
# the apps' lines carry their oracle parity check, which is their cpu_baseline leg
run_app() { timeout 900 python bench.py "$@" 2>/dev/null | tail -1 >> $out; }
run --config 2 --steps 10 --warmup 3
run --config 1 --steps 10 --warmup 3
for d in 1 2 4 8; do run --config 3 --delta $d --steps 10 --warmup 3; done
for d in 1024 4096 16384 32768 65536; do run --config 2 --delta $d --steps 5 --warmup 3 --no-compare; done
run --config 4 --steps 3 --warmup 3 --no-compare
run --config 5 --steps 3 --warmup 3 --no-compare
for c in 1 2 3; do run_app --config $c --app ppsp --steps 10 --warmup 3; done
for c in 1 2; do run_app --config $c --app astar --steps 10 --warmup 3; done
for c in 2 3; do run_app --config $c --app kcore --steps 5 --warmup 3; done
timeout 900 python bench.py --impl reference --config 2 --steps 1 --warmup 0 2>/dev/null | tail -1 >> $out
wc -l $out
