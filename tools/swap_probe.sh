#!/bin/bash
# time hlu_only with alternative builds of libfde.so (dev tool)
for f in "$@"; do
  cp paper_1808_02937_b200/libfde.so /tmp/libfde_orig.so
  cp "$f" paper_1808_02937_b200/libfde.so
  echo "== $f"; FDE_DEBUG_TIMELINE=1 python tools/hlu_only.py 64 2>&1 | grep -v Exception | grep "hlu \|timeline"
  cp /tmp/libfde_orig.so paper_1808_02937_b200/libfde.so
done
