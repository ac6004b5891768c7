#!/bin/bash
# compute-sanitizer on config 1: memcheck / racecheck / synccheck over the smoke
# path (sampler + SEGMENT gather) and the BULK (smem ring + mbarrier) and NAIVE/SHIFT gathers.
for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool: smoke (sampler + segment gather, config 1)"
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python __graft_entry__.py --smoke 2>&1 | tail -4
  echo "=== $tool: gather variants"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/workers/san_variants.py 2>&1 | tail -4
done
