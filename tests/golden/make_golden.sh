#!/bin/sh
# Regenerates tests/golden/trainer_*.json from the UNMODIFIED reference
# (needs /root/reference; run in the build container, not on the GPU box).
set -e
here=$(cd "$(dirname "$0")" && pwd)
make -s -C "$here/../../oracle" ref
"$here/../../oracle/_ref/gen_golden" "$here"
