#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python tools/gather_probe.py > gpurun_out/r02d_gather.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_ltcfabric.sum --clock-control none -k regex:gather -c 24 --csv --log-file gpurun_out/r02d_ncu.csv python tools/gather_probe.py > gpurun_out/r02d_ncu.log 2>&1
