#!/bin/bash
# Round-2 GPU runs, one arm per gpurun call of the round (each arm was a tools/run_r02<arm>.sh
# script before they were folded here). Usage on the GPU box:
#   bash tools/r02_runs.sh ARM [args]      (outputs under gpurun_out/, summaries in profiles/)
# Variant libraries for the A/B arms are built here first with tools/ab_build.sh (AB_OUT=tools/abx).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
arm=$1; shift
case $arm in
  aa)  # round 2 (session 4): k-core — slot path without the warp match + evict-first slots (now default), packed 4-byte edges on the CSR path (GI_KC_PACK=0: the 8-byte edges); k-core parity tests
export AB_DIR=abm AB_ONLY=main
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "kcore" > gpurun_out/r02aa_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02aa_tests.log
tail -2 gpurun_out/r02aa_tests.log
for r in 1 2; do for pk in 1 0; do
  GI_KC_PACK=$pk timeout 600 python tools/ab_kcore.py 3 2>&1 | grep libgi | sed "s/^/cfg 3 pack=$pk: /" >> gpurun_out/r02aa_ab.log
done; done
timeout 600 python tools/ab_kcore.py 2 2>&1 | grep libgi | sed "s/^/cfg 2: /" >> gpurun_out/r02aa_ab.log
;;
  ab)  # round 2 (session 4): extraction dist reads with an L2 evict-first policy (A/B on configs 4 and 3)
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in xd0 xd1; do
  for cd in "4 2" "3 2" "2 65536"; do AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02ab_ab.log; done
done; done
;;
  ac)  # round 2 (session 4): the persistent kernel's pre-reads through the expand mirror — tests, A/B
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window or mirror or split or expand or stress or ppsp or astar or hubs" > gpurun_out/r02ac_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ac_tests.log
tail -2 gpurun_out/r02ac_tests.log
for r in 1 2; do for v in pm0 pm1; do
  AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4: /" >> gpurun_out/r02ac_ab.log
done; done
;;
  ae)  # round 2 (session 4): the bucket window opened late (GI_WINDOW_PILE) — tests, config 4 A/B
export GI_GEN_CACHE=/tmp/gcache
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window" > gpurun_out/r02ae_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ae_tests.log
tail -2 gpurun_out/r02ae_tests.log
for r in 1 2; do for wp in "0 0" "4 2000000" "4 8000000" "8 4000000" "2 1000000"; do
  set -- $wp
  GI_WINDOW=$1 GI_WINDOW_PILE=$2 timeout 600 python tools/time_cfg.py 4 2 '{}' 2>&1 | grep ms_median | cut -c1-330 | sed "s/^/window=$1 pile=$2 /" >> gpurun_out/r02ae_ab.log
done; done
;;
  af)  # round 2 (session 4): fusion threshold T on config 4 (expand query)
export GI_GEN_CACHE=/tmp/gcache
for r in 1 2; do
  timeout 900 python tools/time_cfg.py 4 2 '{}' '{"threshold": 16}' '{"threshold": 64}' '{"threshold": 1024}' '{"threshold": 4096}' '{"fusion": false}' 2>&1 | grep ms_median | cut -c1-260 >> gpurun_out/r02af_T4.log
done
;;
  b)  # GPU tests after the cluster-flag fix, the fusion-threshold sweep and the eager/lazy table
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02b_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02b_tests.log
timeout 900 python tools/sweep_T.py 1 2 3 > gpurun_out/r02b_sweepT.md 2>&1
timeout 900 python tools/lazy_table.py 1 2 3 4 > gpurun_out/r02b_lazy.md 2>&1
;;
  c)  # round-2 (session 2) check: GPU tests, default bench, config-4 launch list with DRAM bytes
export GI_GEN_CACHE=/tmp/gcache
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02c_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02c_tests.log
( time timeout 1500 python bench.py ) > gpurun_out/r02c_bench.log 2> gpurun_out/r02c_bench.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary --no-compare"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand" --csv --log-file gpurun_out/r02c_launches.csv $CMD > gpurun_out/r02c_ncu1.log 2>&1
;;
  d)  # traces of config 4 (1024 threads) and config 2 (512), and the config-5 batch Δ / shape sweep
export GI_GEN_CACHE=/tmp/gcache
TRACE_W=1024 TRACE_SO=tools/ab/libgi_trace1024.so timeout 600 python tools/trace_async.py cfg4 2 bsp > gpurun_out/r02d_trace_cfg4.log 2>&1
TRACE_W=512 TRACE_SO=tools/ab/libgi_trace512.so timeout 600 python tools/trace_async.py cfg2 65536 bsp > gpurun_out/r02d_trace_cfg2.log 2>&1
timeout 900 python tools/batch_sweep.py 4096,8192,16384,32768,65536 '{}' > gpurun_out/r02d_batch_delta.log 2>&1
timeout 600 python tools/batch_sweep.py 8192 '{"cta_threads": 512}' '{"group_ctas": 4, "cta_threads": 512}' '{"rung": 3}' > gpurun_out/r02d_batch_shape.log 2>&1
;;
  e)  # traces of config 4 (fused and unfused, 1024-thread trace build) and config 4 fusion thresholds
export GI_GEN_CACHE=/tmp/gcache
TRACE_W=1024 TRACE_SO=tools/ab/libgi_trace1024.so timeout 600 python tools/trace_async.py cfg4 2 bsp > gpurun_out/r02e_trace_cfg4.log 2>&1
TRACE_W=1024 TRACE_SO=tools/ab/libgi_trace1024.so timeout 600 python tools/trace_async.py cfg4 2 unfused > gpurun_out/r02e_trace_cfg4u.log 2>&1
timeout 900 python tools/time_cfg.py 4 2 '{}' '{"fusion": false}' '{"threshold": 64}' '{"threshold": 1024}' '{"threshold": 2048}' > gpurun_out/r02e_cfg4_T.log 2>&1
;;
  f)  # extraction split: parity (new test + split tests + config 4 full), timing on config 4
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "extract_split or expand_split or expand_edge or hand_examples or lazy or config3_full" > gpurun_out/r02f_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02f_tests.log
timeout 900 python tools/time_cfg.py 4 2 '{}' '{"fusion": false}' '{"threshold": 1024}' > gpurun_out/r02f_cfg4.log 2>&1
GI_XSPLIT_MIN=0 timeout 600 python tools/time_cfg.py 4 2 '{}' > gpurun_out/r02f_cfg4_nox.log 2>&1
GI_XSPLIT_MIN=500000 timeout 600 python tools/time_cfg.py 4 2 '{}' > gpurun_out/r02f_cfg4_x500k.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config4_full" > gpurun_out/r02f_cfg4_parity.log 2>&1
echo "rc=$?" >> gpurun_out/r02f_cfg4_parity.log
;;
  g)  # k-core slot path vs CSR path on configs 1-3 (tests + timings), config-4 launch list
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "kcore" > gpurun_out/r02g_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02g_tests.log
for c in 2 3 1; do
  timeout 300 python tools/profile_run.py --config $c --kcore --reps 5 > gpurun_out/r02g_kc$c.log 2>&1
  GI_KC_SLOTS=0 timeout 300 python tools/profile_run.py --config $c --kcore --reps 5 > gpurun_out/r02g_kc${c}_csr.log 2>&1
done
timeout 300 python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02g_plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand|extract" --csv --log-file gpurun_out/r02g_launches4.csv python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02g_ncu4.log 2>&1
;;
  h)  # L1-cached expand pre-reads (variant l1) vs base on configs 4 and 3
export GI_GEN_CACHE=/tmp/gcache
for r in 1 2; do for v in base l1; do
  AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 >> gpurun_out/r02h_ab4.log 2>&1
done; done
for v in base l1; do AB_ONLY=$v timeout 600 python tools/ab_time.py 3 2 >> gpurun_out/r02h_ab3.log 2>&1; done
;;
  m)  # round 2 (session 4): expand's mirror filter — parity of the split paths, then config 4 A/B
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mirror or split or expand" > gpurun_out/r02m_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02m_tests.log
for r in 1 2; do for mv in 1 0; do
  GI_MIRROR=$mv timeout 600 python tools/time_cfg.py 4 2 '{}' >> gpurun_out/r02m_ab4.log 2>&1; echo "mirror=$mv" >> gpurun_out/r02m_ab4.log
done; done
;;
  n)  # round 2 (session 4): mirror test, config-4 launch list with DRAM bytes (mirror on), config-2 level trace
export GI_GEN_CACHE=/tmp/gcache
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mirror" > gpurun_out/r02n_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02n_tests.log
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02n_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand|extract" --csv --log-file gpurun_out/r02n_launches.csv python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02n_ncu1.log 2>&1
TRACE_W=512 timeout 900 python tools/trace_async.py cfg2 65536 bsp > gpurun_out/r02n_trace_cfg2.log 2>&1
;;
  o)  # round 2 (session 4): stage-A warp skip A/B (tools/abx/libgi_{base,wskip}.so) and the finer cfg2 level trace
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
TRACE_W=512 TRACE_SO=$GRAFT_REPO_ROOT/tools/abx/libgi_trace512.so timeout 600 python tools/trace_async.py cfg2 65536 bsp > gpurun_out/r02o_trace_cfg2.log 2>&1
for r in 1 2; do for v in base wskip; do
  for cd in "2 65536" "1 1000" "3 2" "5 8192"; do
    AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02o_ab.log
  done
done; done
for v in base wskip; do AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4: /" >> gpurun_out/r02o_ab.log; done
;;
  p)  # round 2 (session 4): L2 policies for the wavefront's dist lines vs the slot stream (A/B)
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in base el ef elef persist; do
  for cd in "2 65536" "1 1000" "5 8192" "3 2"; do
    if [ $v = persist ]; then
      GI_L2_PERSIST=1 AB_ONLY=base timeout 600 python tools/ab_time.py $cd 2>&1 | grep -E "libgi|L2 window" | sed "s/^/cfg $cd persist: /" >> gpurun_out/r02p_ab.log
    else
      AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02p_ab.log
    fi
  done
done; done
;;
  q)  # round 2 (session 4): expand fast block path + 32-bit edge positions (A/B on config 4), split-path parity
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mirror or split or expand" > gpurun_out/r02q_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02q_tests.log
for r in 1 2; do
  GI_IDX32=0 AB_ONLY=fb0 timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg4 fb0 idx64: /" >> gpurun_out/r02q_ab.log
  AB_ONLY=fb0 timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg4 fb0 idx32: /" >> gpurun_out/r02q_ab.log
  AB_ONLY=fb1 timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg4 fb1 idx32: /" >> gpurun_out/r02q_ab.log
done
;;
  r)  # round 2 (session 4): bucket window — parity of the split/window paths, then config 4 per width
export GI_GEN_CACHE=/tmp/gcache
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window or mirror or split or expand" > gpurun_out/r02r_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02r_tests.log
tail -3 gpurun_out/r02r_tests.log
for r in 1 2; do for w in 0 4 8 16; do
  GI_WINDOW=$w timeout 600 python tools/time_cfg.py 4 2 '{}' 2>&1 | grep ms_median | sed "s/^/window=$w /" >> gpurun_out/r02r_ab4.log
done; done
;;
  s)  # round 2 (session 4): slot-load L2 policy A/B on every config (c0 = the mirror commit's build)
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in c0 ef0 ef1; do
  for cd in "4 2" "2 65536" "5 8192" "3 2"; do
    AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02s_ab.log
  done
done; done
;;
  t)  # round 2 (session 4) evidence run: full GPU tests, default bench (config 4 headline), reference arm, the config-4 launch list with DRAM bytes, then configs 1-3, 5 and the apps
T=${1:-r02t}
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
;;
  u)  # round 2 (session 4): expand rows-in-flight sweep (kXRows) with the mirror, and a --set full capture of config 4's hub-phase expand_kernel (the second expand launch of the query)
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in xr4 xr8 xr12 xr16; do
  AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg4: /" >> gpurun_out/r02u_ab.log
done; done
ncu --set full --clock-control none --import-source on -k regex:expand_kernel -s 1 -c 1 -o gpurun_out/r02u_expand -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02u_ncu.log 2>&1
;;
  v)  # round 2 (session 4): batched host segment loop (speculative [expand, extract, resume] rounds)
export GI_GEN_CACHE=/tmp/gcache
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window or mirror or split or expand or ppsp or astar or stress" > gpurun_out/r02v_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02v_tests.log
tail -3 gpurun_out/r02v_tests.log
for r in 1 2 3; do timeout 600 python tools/time_cfg.py 4 2 '{}' '{"fusion": false}' 2>&1 | grep ms_median | cut -c1-300 >> gpurun_out/r02v_cfg4.log; done
;;
  w)  # round 2 (session 4): config-5 batch group shapes (CTAs per group, threads per CTA, rung) at Δ=2^13
timeout 1500 python tools/batch_sweep.py 8192 '{}' '{"group_ctas": 1}' '{"group_ctas": 2}' '{"group_ctas": 4}' \
  '{"group_ctas": 2, "cta_threads": 512}' '{"group_ctas": 4, "cta_threads": 512}' '{"group_ctas": 1, "cta_threads": 512}' \
  '{"group_ctas": 2, "threshold": 4096}' '{"group_ctas": 2, "threshold": 1024}' '{"group_ctas": 2, "rung": "grid"}' > gpurun_out/r02w_batch.log 2>&1
;;
  x)  # round 2 (session 4): the parent-edge skip of the low-degree fused kernels — GPU tests, then A/B
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
GI_SKIP_CFG4=1 timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r02x_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02x_tests.log
tail -3 gpurun_out/r02x_tests.log
for r in 1 2; do for v in par0 par1; do
  for cd in "2 65536" "1 1000" "5 8192" "2 16384"; do
    AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02x_ab.log
  done
done; done
;;
  y)  # round 2 (session 4): --set full captures of config 4's persistent segments (the post-hub-phase segment and the tail segment) for the stall and traffic breakdown
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02y_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sssp_persistent -s 5 -c 1 -o gpurun_out/r02y_seg5 -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02y_ncu5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sssp_persistent -s 17 -c 1 -o gpurun_out/r02y_seg17 -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02y_ncu17.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:extract_kernel -s 1 -c 1 -o gpurun_out/r02y_extract -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02y_ncux.log 2>&1
;;
  z)  # round 2 (session 4): k-core slot path — warp match vs one atomic per edge, slot evict-first (A/B)
export AB_DIR=abx
for r in 1 2; do for v in kb knm kef knmef; do
  for c in 2 1; do AB_ONLY=$v timeout 600 python tools/ab_kcore.py $c 2>&1 | grep libgi | sed "s/^/cfg $c: /" >> gpurun_out/r02z_ab.log; done
done; done
;;
  all)  # round-2 full run: GPU tests, the default bench (no generator cache, as the driver runs it), the reference arm, and the secondary app lines. Usage: run_all_r02.sh [tag] (default r02aj)
T=${1:-r02aj}
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${T}_tests.log
( time timeout 1500 python bench.py ) > gpurun_out/${T}_bench.log 2> gpurun_out/${T}_bench.err
( time timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/${T}_ref.log 2> gpurun_out/${T}_ref.err
for c in 1 2 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3; done > gpurun_out/${T}_cfgs.log 2>&1
timeout 900 python bench.py --config 5 --steps 5 --warmup 2 > gpurun_out/${T}_cfg5.log 2>&1
for app in ppsp astar kcore; do timeout 600 python bench.py --config 2 --app $app --steps 10 --warmup 3; done > gpurun_out/${T}_apps.log 2>&1
timeout 600 python bench.py --config 3 --app kcore --steps 10 --warmup 3 >> gpurun_out/${T}_apps.log 2>&1
;;
  profile_cfg4)  # round-2 profiles of the config-4 headline: the bench launch list (time + DRAM bytes per launch), then ncu --set full of the hub-phase expand_kernel and the heaviest persistent segment
export GI_GEN_CACHE=/tmp/gcache
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary --no-compare"
$CMD > gpurun_out/r02ad_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand" --csv --log-file gpurun_out/r02ad_launches.csv $CMD > gpurun_out/r02ad_ncu1.log 2>&1
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02ad_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:expand_kernel -s 1 -c 1 -o gpurun_out/r02ad_expand -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02ad_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sssp_persistent -s 3 -c 1 -o gpurun_out/r02ad_persist -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02ad_ncu3.log 2>&1
;;
  rung)  # execution-group rungs (CTA / cluster / grid) on configs 1, 2, 3 and the config-5 batch
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "rungs or hand or path or capi" > gpurun_out/rung_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rung_tests.log
timeout 600 python tools/time_cfg.py 1 1000 '{}' '{"rung": "cta"}' '{"rung": "cluster", "group_ctas": 4}' '{"rung": "cluster", "group_ctas": 8}' '{"rung": "cluster", "group_ctas": 16}' '{"max_ctas": 16}' > gpurun_out/rung_time1.log 2>&1
timeout 600 python tools/time_cfg.py 2 65536 '{}' '{"rung": "cluster", "group_ctas": 16}' > gpurun_out/rung_time2.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"rung": "cluster", "group_ctas": 16}' > gpurun_out/rung_time3.log 2>&1
timeout 900 python - > gpurun_out/rung_time5.log 2>&1 <<'PY'
import sys, json, statistics; sys.path.insert(0, '.')
import torch, gen
from paper_1911_07260_b200 import gi
g = gen.config_graph(5); G = gi.Graph.from_csr(g); srcs = gen.config_sources(5, g, 64)
out = torch.empty((64, g.n), dtype=torch.int32, device="cuda")
for o in ({}, {"rung": "cta"}, {"rung": "cluster", "group_ctas": 2}, {"rung": "cluster", "group_ctas": 4}, {"group_ctas": 4}):
    ts = []
    for i in range(3):
        st = gi.gi_sssp_batch(G, srcs, 8192, out, gi.make_options(**o)); ts.append(st[0].gpu_ms)
    print(json.dumps({"opts": o, "ms": statistics.median(ts), "groups": st[0].groups, "ctas": st[0].ctas, "rung": st[0].rung}), flush=True)
PY
;;
  ag)  # expand rows with no candidate past the mirror skip the atomics and pushes (GI_X_XSKIP) — tests, config 4 A/B
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window or mirror or split or expand" > gpurun_out/r02ag_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ag_tests.log
tail -2 gpurun_out/r02ag_tests.log
for r in 1 2 3; do for v in xs0 xs1; do
AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4: /" >> gpurun_out/r02ag_ab.log
done; done
;;
  ah)  # expand: a block's candidates past the mirror compacted and relaxed densely (GI_X_XCOMPACT) — tests, config 4 A/B
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window or mirror or split or expand or stress or hubs" > gpurun_out/r02ah_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ah_tests.log
tail -2 gpurun_out/r02ah_tests.log
for r in 1 2 3; do for v in xc0 xc1; do
AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4: /" >> gpurun_out/r02ah_ab.log
done; done
;;
  ai)  # expand: a block inside one list entry mapped once (GI_X_FASTBLK), after the compaction — config 4 A/B
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2 3; do for v in fb0 fb1; do
AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4: /" >> gpurun_out/r02ai_ab.log
done; done
;;
  aj)  # relax_batch: warps with no lowering after the pre-read / mirror filter skip the pushes (GI_X_RSKIP) — tests, A/B
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config3 or hubs or split or expand or mirror or stress or astar" > gpurun_out/r02aj_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02aj_tests.log
tail -2 gpurun_out/r02aj_tests.log
for r in 1 2 3; do for v in rs0 rs1; do
for cd in "4 2" "3 2"; do AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02aj_ab.log; done
done; done
;;
  ak)  # ncu --set full of config 4's hub-phase expand_kernel after the vote-skip and compaction
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02ak_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:expand_kernel -s 1 -c 1 -o gpurun_out/r02ak_expand -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02ak_ncu.log 2>&1
;;
  al)  # config-5 batch: pre-read on, async drain, unfused (option sweep at Δ=2^13)
timeout 1500 python tools/batch_sweep.py 8192 '{}' '{"pre_read": 1}' '{"drain": "async"}' '{"fusion": false}' '{"pre_read": 1, "group_ctas": 4}' > gpurun_out/r02al_batch.log 2>&1
;;
  am)  # expand: one window-coverage test per block (GI_X_WCOVER) — split/expand tests, config 4 A/B
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window or mirror or split or expand" > gpurun_out/r02am_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02am_tests.log
tail -2 gpurun_out/r02am_tests.log
for r in 1 2 3; do for v in wc0 wc1; do
AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4: /" >> gpurun_out/r02am_ab.log
done; done
;;
  an)  # round 2 (session 5): evidence run at HEAD from the re-created container, config-4 parity JSON, config-5 chain-vs-work probe
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02an_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02an_tests.log
( time timeout 1500 python bench.py ) > gpurun_out/r02an_bench.log 2> gpurun_out/r02an_bench.err
timeout 600 python tools/batch_ecc.py > gpurun_out/r02an_batch_ecc.log 2>&1
timeout 1500 python tests/run_cfg4.py --reps 2 > gpurun_out/r02an_cfg4_parity.json 2> gpurun_out/r02an_cfg4_parity.err
;;
  ao)  # round 2 (session 5): slot prefetches of big extractions' live vertices (GI_X_PFX, GI_X_PFAGG) and extract_kernel at 4 entries per thread, 2 CTAs per SM (e4) — config 4 / 3 A/B
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2 3; do for v in pf11 pf01 pf00 e4; do
AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4: /" >> gpurun_out/r02ao_ab.log
done; done
for v in pf11 pf01 pf00 e4; do
AB_ONLY=$v timeout 600 python tools/ab_time.py 3 2 2>&1 | grep libgi | sed "s/^/cfg 3: /" >> gpurun_out/r02ao_ab.log
done
;;
  ap)  # round 2 (session 5): big-extraction slot prefetches off (new default, "old" = on); expand's current-bucket (xc0) and the global-frontier (pg0) prefetches — A/B on configs 4, 3, 2, 5, then the GPU tests
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in base old xc0 pg0; do
AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4: /" >> gpurun_out/r02ap_ab.log
done; done
for cd in "3 2" "2 65536" "5 8192"; do for v in base old xc0 pg0; do
AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02ap_ab.log
done; done
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02ap_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ap_tests.log
;;
  aq)  # round 2 (session 5): evidence after the prefetch change — default bench, config-4 launch list with DRAM bytes, configs 1-3, 5 and the apps; k-core prefetch A/B
T=${1:-r02aq}
( time timeout 1500 python bench.py ) > gpurun_out/${T}_bench.log 2> gpurun_out/${T}_bench.err
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/${T}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand|extract" --csv --log-file gpurun_out/${T}_launches_cfg4.csv python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/${T}_ncu1.log 2>&1
for c in 1 2 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3; done > gpurun_out/${T}_cfgs.log 2>&1
timeout 900 python bench.py --config 5 --steps 5 --warmup 2 > gpurun_out/${T}_cfg5.log 2>&1
for app in ppsp astar kcore; do timeout 600 python bench.py --config 2 --app $app --steps 10 --warmup 3; done > gpurun_out/${T}_apps.log 2>&1
timeout 600 python bench.py --config 3 --app kcore --steps 10 --warmup 3 >> gpurun_out/${T}_apps.log 2>&1
# k-core slot prefetch only for vertices kept below T in the CTA's bin (GI_KC_PFLOCAL: kpf1) vs every finished vertex (kpf0)
for r in 1 2; do for v in kpf0 kpf1; do for c in 2 3; do
AB_DIR=abk AB_ONLY=$v timeout 600 python tools/ab_kcore.py $c 2>&1 | grep libgi | sed "s/^/cfg $c: /" >> gpurun_out/${T}_kcore_ab.log
done; done; done
;;
  ar)  # round 2 (session 5): the init's Dist = {inf} stores with the streaming hint (GI_INIT_CS: ics1) vs plain (ics0) — A/B on configs 5, 4, 2, 3
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in ics0 ics1; do for cd in "5 8192" "4 2"; do
AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02ar_ab.log
done; done; done
for v in ics0 ics1; do for cd in "2 65536" "3 2"; do
AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02ar_ab.log
done; done
# the GPU tests with the new defaults (k-core GI_KC_PFLOCAL=1, expand GI_X_PFXC=0)
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02ar_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ar_tests.log
;;
  as)  # round 2 (session 5): k-core app lines with GI_KC_PFLOCAL=1, and ncu --set full of config 2's persistent kernel and of config 2's k-core kernel at the final build
export GI_GEN_CACHE=/tmp/gcache
for c in 2 3; do timeout 600 python bench.py --config $c --app kcore --steps 10 --warmup 3; done > gpurun_out/r02as_apps.log 2>&1
python tools/profile_run.py --config 2 --delta 65536 --reps 1 > gpurun_out/r02as_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:sssp_persistent -c 1 -o gpurun_out/r02as_cfg2 -f python tools/profile_run.py --config 2 --delta 65536 --reps 1 > gpurun_out/r02as_ncu.log 2>&1
python tools/profile_run.py --config 2 --kcore --reps 1 > gpurun_out/r02as_kplain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:kcore_persistent -c 1 -o gpurun_out/r02as_kcore2 -f python tools/profile_run.py --config 2 --kcore --reps 1 > gpurun_out/r02as_kncu.log 2>&1
;;
  at)  # round 2 (session 5): slot prefetches of small in-kernel extractions (xs0: off) and of every global-frontier push too (np) — A/B on configs 5, 2, 3, 4
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in base xs0 np; do for cd in "5 8192" "2 65536"; do
AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02at_ab.log
done; done; done
for v in base xs0 np; do for cd in "3 2" "4 2" "1 1000"; do
AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02at_ab.log
done; done
;;
  au)  # round 2 (session 5): final evidence — GPU tests at the final defaults (all big-list slot prefetches off), default bench, config-4 launch list with DRAM bytes, configs 2, 3, 5
T=${1:-r02au}
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${T}_tests.log
( time timeout 1500 python bench.py ) > gpurun_out/${T}_bench.log 2> gpurun_out/${T}_bench.err
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/${T}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand|extract" --csv --log-file gpurun_out/${T}_launches_cfg4.csv python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/${T}_ncu1.log 2>&1
for c in 2 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3; done > gpurun_out/${T}_cfgs.log 2>&1
timeout 900 python bench.py --config 5 --steps 5 --warmup 2 > gpurun_out/${T}_cfg5.log 2>&1
;;
  av)  # round 2 (session 6): ncu --set full of config 4's hub-phase expand_kernel at the final build (all big-list slot prefetches off), then the app lines
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02av_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:expand_kernel -s 1 -c 1 -o gpurun_out/r02av_expand -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02av_ncu.log 2>&1
for app in ppsp astar kcore; do timeout 600 python bench.py --config 2 --app $app --steps 10 --warmup 3; done > gpurun_out/r02av_apps.log 2>&1
timeout 600 python bench.py --config 3 --app kcore --steps 10 --warmup 3 >> gpurun_out/r02av_apps.log 2>&1
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/r02av_cfg1.log 2>&1
;;
  aw)  # round 2 (session 6): race soak at the final build — the full-size stress test with 4 more seeds x 40 runs per leg, two of them with every expand / extraction split into its own kernels (GI_SPLIT_MIN=1, GI_XSPLIT_MIN=1)
export GI_GEN_CACHE=/tmp/gcache GI_STRESS_ITERS=40
for seed in 11 12 13 14; do
  if [ $seed -ge 13 ]; then export GI_SPLIT_MIN=1 GI_XSPLIT_MIN=1; fi
  echo "== seed $seed iters $GI_STRESS_ITERS split_min=${GI_SPLIT_MIN:-default}" >> gpurun_out/r02aw_soak.log
  GI_STRESS_SEED=$seed timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "stress_repeated" >> gpurun_out/r02aw_soak.log 2>&1
  echo "rc=$?" >> gpurun_out/r02aw_soak.log
done
;;
  ax)  # round 2 (session 6): expand rows in flight per warp re-swept at the final build (GI_XROWS 6 / 8 = base / 10) — config 4 A/B, three alternating rounds
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2 3; do for v in base xr6 xr10; do
AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4 2: /" >> gpurun_out/r02ax_ab.log
done; done
;;
  ay)  # round 2 (session 6): the config-4 placement effect re-measured at the final build (tools/placement_test.py, tools/ab/libgi_cs.so = the default build), one mode per process
export GI_GEN_CACHE=/tmp/gcache
for m in single torch_mb_256 out_first torch_mb_256_free torch_mb_2048 single torch_mb_256; do
timeout 600 python tools/placement_test.py $m 2>&1 | tail -1 >> gpurun_out/r02ay_placement.log
done
;;
  az)  # round 2 (session 6): DRAM bytes per query of configs 2, 3 and 5 at the final build (ncu metrics-only launch lists → profiles/ncu_traffic.json)
export GI_GEN_CACHE=/tmp/gcache
for cd in "2 65536" "3 2" "5 8192"; do set -- $cd
python tools/profile_run.py --config $1 --delta $2 --reps 1 > gpurun_out/r02az_plain_cfg$1.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand|extract" --csv --log-file gpurun_out/r02az_launches_cfg$1.csv python tools/profile_run.py --config $1 --delta $2 --reps 1 > gpurun_out/r02az_ncu_cfg$1.log 2>&1
done
;;
  *) echo "usage: bash tools/r02_runs.sh ARM [args]; arms:"; grep -E "^  [a-z0-9_]+\)" "$0"; exit 2 ;;
esac
