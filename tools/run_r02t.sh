#!/bin/bash
# round 2 (session 4) evidence run: full GPU tests, default bench (config 4 headline), reference arm,
# the config-4 launch list with DRAM bytes, then configs 1-3, 5 and the apps
T=${1:-r02t}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${T}_tests.log
( time timeout 1500 python bench.py ) > gpurun_out/${T}_bench.log 2> gpurun_out/${T}_bench.err
( time timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/${T}_ref.log 2> gpurun_out/${T}_ref.err
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/${T}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand|extract" --csv --log-file gpurun_out/${T}_launches_cfg4.csv python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/${T}_ncu1.log 2>&1
for c in 1 2 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3; done > gpurun_out/${T}_cfgs.log 2>&1
timeout 900 python bench.py --config 5 --steps 5 --warmup 2 > gpurun_out/${T}_cfg5.log 2>&1
for app in ppsp astar kcore; do timeout 600 python bench.py --config 2 --app $app --steps 10 --warmup 3; done > gpurun_out/${T}_apps.log 2>&1
timeout 600 python bench.py --config 3 --app kcore --steps 10 --warmup 3 >> gpurun_out/${T}_apps.log 2>&1
