#!/bin/bash
# Build the library as it is in the working tree into build/variants/<name>.so
# (for same-box A/B runs with ST_LIB_VARIANT=...). Usage: tools/build_variant.sh <name>
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=${1:?name}
mkdir -p $ROOT/build/variants
make -s -j16 -C $ROOT/paper_2305_09781_b200/csrc
cp $ROOT/paper_2305_09781_b200/libspectree_b200.so $ROOT/build/variants/$NAME.so
echo "built $ROOT/build/variants/$NAME.so"
