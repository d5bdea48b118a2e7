#!/bin/bash
# EPG-RB on C3 / C4 with the bitset frontier (new) against the heap frontier (base): phase times
mkdir -p gpurun_out
for v in base new base new; do
  if [ $v = new ]; then unset EPG_LIB_PATH; else export EPG_LIB_PATH=$PWD/tools/_trace/libepg_base.so; fi
  echo "== $v" >> gpurun_out/r3r_rb.err
  EPG_RB_TRACE=1 timeout 900 python tools/partition_bench.py c3 --leaf-parts 2048 >> gpurun_out/r3r_rb_$v.jsonl 2>> gpurun_out/r3r_rb.err
done
