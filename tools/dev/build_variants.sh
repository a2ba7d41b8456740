#!/bin/bash
# DEV: build libgmg.so once per set of -D defines into tools/dev/so/libgmg_<name>.so
# usage: tools/dev/build_variants.sh name1 "-DA -DB" name2 "-DC" ...
set -e
cd "$(dirname "$0")/../.."
while [ $# -ge 2 ]; do
    GMG_NVCC_DEFS="$2" python -c "from paper_2509_06347_b200 import _build; _build.build(force=True)" 2>/dev/null
    cp paper_2509_06347_b200/libgmg.so tools/dev/so/libgmg_$1.so
    echo "built $1: $2"
    shift 2
done
python -c "from paper_2509_06347_b200 import _build; _build.build(force=True)" 2>/dev/null
