#!/bin/bash
# DRAM read/write split and L2 sector requests per launch of the cfg2 VNR decode
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read.sum \
    --clock-control none -k regex:"k_check" --csv --log-file gpurun_out/lm2.csv python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/ncu_lm2.log 2>&1
echo "ncu=$?"
