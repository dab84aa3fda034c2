#!/bin/bash
# A/B timing on the GPU box: alternates library builds / env settings over tools/sweep.py.
#   tools/ab_session.sh OUT "cfg1 cfg2 ..." variant1 variant2 ...
# variant = LIB[@VAR=VAL[,VAR=VAL...]]; LIB "cur" = the in-tree library, others =
# tools/_build/<LIB>/libmcmi.so
out=$1; shift; cfgs=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    lib=${v%%@*}; envs=""; [[ "$v" == *@* ]] && envs=${v#*@}
    if [ "$lib" = cur ]; then unset MCMI_LIB_PATH; else export MCMI_LIB_PATH=tools/_build/$lib/libmcmi.so; fi
    echo "== $v"
    env ${envs//,/ } timeout 600 python tools/sweep.py $cfgs
  done
done > "$out" 2>&1
unset MCMI_LIB_PATH
python tools/ab.py report "$out"
