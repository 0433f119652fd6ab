#!/bin/bash
# usage: tools/run_variants.sh name... : prof_step.py under each build/variants/libfgtcuda_<name>.so
for v in "$@"; do
  echo "== $v"
  FGT_LIB_PATH=build/variants/libfgtcuda_$v.so python tools/prof_step.py 2>&1 | tail -1 | cut -c1-200
done
