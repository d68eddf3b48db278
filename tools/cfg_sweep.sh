#!/bin/bash
# tools/cfg_sweep.sh WORKLOAD LIB... : device-resident ms/step per experiment library
wl=$1; shift
BENCH_ARGS="--workload $wl" bash tools/lib_sweep.sh "$@" | sed "s/^/$wl /"
