#!/bin/bash
# compute-sanitizer over the session-2 paths (tests/workers/san_s2.py) and the smoke path.
for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool: smoke (sampler + segment gather, config 1)"
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python __graft_entry__.py --smoke 2>&1 | tail -3
  echo "=== $tool: zero-copy CSR, launch shapes, hints, cached gather"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/workers/san_s2.py 2>&1 | tail -3
done
