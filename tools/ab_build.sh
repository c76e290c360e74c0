#!/bin/bash
# Build the committed (HEAD) library into _ab/libcerdot_head.so for A/B timing against the working tree
# (select with CERDOT_LIB=...).  Usage: tools/ab_build.sh
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/cerdot_ab && mkdir -p /tmp/cerdot_ab _ab
git archive HEAD paper_1805_10692_b200 include | tar -x -C /tmp/cerdot_ab
(cd /tmp/cerdot_ab && python -m paper_1805_10692_b200.build --force >/dev/null)
cp /tmp/cerdot_ab/paper_1805_10692_b200/_lib/libcerdot.so _ab/libcerdot_head.so
echo _ab/libcerdot_head.so
