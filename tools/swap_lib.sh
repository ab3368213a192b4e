#!/bin/bash
# run a command with an alternative libdk.so (experiment builds); restores the original after
set -e
cp paper_1510_02148_b200/_lib/libdk.so /tmp/libdk_orig.so
cp "$1" paper_1510_02148_b200/_lib/libdk.so
shift
"$@" || true
cp /tmp/libdk_orig.so paper_1510_02148_b200/_lib/libdk.so
