#!/bin/bash
# Build librpd of a git revision (default HEAD) into paper_2403_18761_b200/librpd_head.so, for
# in-process A/B timing with tools/ab.py (tag:@paper_2403_18761_b200/librpd_head.so).
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2403_18761_b200/csrc include | tar -x -C "$TMP"
cd "$TMP"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -I include -o "$ROOT/paper_2403_18761_b200/librpd_head.so" \
  paper_2403_18761_b200/csrc/*.cu
rm -rf "$TMP"
