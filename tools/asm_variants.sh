#!/bin/bash
# Development tool: time the BEM assembly kernels of several prebuilt library
# variants (variants/lib_v*.so, each a full libfdsweep_b200.so) on the GPU box,
# with the assembly parity tests run against each.
set -u
cp paper_1511_04355_b200/libfdsweep_b200.so /tmp/lib_head.so
for v in variants/lib_v*.so; do
  cp "$v" paper_1511_04355_b200/libfdsweep_b200.so
  echo "== $v"
  python tools/perf_asm.py
  python tools/perf_asm.py
  python -m pytest tests/test_gpu_bem.py -q -x -k "parity" 2>&1 | tail -2
done
cp /tmp/lib_head.so paper_1511_04355_b200/libfdsweep_b200.so
