#!/bin/bash
# DEV (on the GPU box): time tools/sweep_variants.py once per prebuilt variant library, in the given order
cd "$(dirname "$0")/../.."
cp paper_2509_06347_b200/libgmg.so /tmp/libgmg_keep.so
for v in "$@"; do
    cp tools/dev/so/libgmg_$v.so paper_2509_06347_b200/libgmg.so
    LANES=0 python ${TIMER:-tools/sweep_variants.py} 2>&1 | tail -1 | sed "s/^/$v /"
done
cp /tmp/libgmg_keep.so paper_2509_06347_b200/libgmg.so
