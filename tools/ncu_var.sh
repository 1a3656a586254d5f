#!/bin/bash
# ncu --set full of a build variant on the config-3 batch: bash tools/ncu_var.sh VARIANT PREC
cd $GRAFT_REPO_ROOT
export TOR_B200_LIB=variants/lib_$1.so
timeout 300 python tools/cfg3_once.py $2 > gpurun_out/var_$1_plain.log 2>&1 || exit 1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:subtree -s 1 -c 1 -o gpurun_out/var_$1 python tools/cfg3_once.py $2 > gpurun_out/var_$1_ncu.log 2>&1
echo "ncu exit $?"
