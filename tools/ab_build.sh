#!/bin/bash
# Build an A/B variant of libdgsip.so with extra defines into build_ab/lib<NAME>.so
#   tools/ab_build.sh NAME "-DFOO=1 -DBAR" [PSET]
set -e
NAME=$1; DEFS=$2; PSET=${3:-0x20}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/ab_$NAME
rm -rf $T && mkdir -p $T
cp -r $ROOT/paper_2112_04167_b200 $ROOT/include $T/
rm -rf $T/paper_2112_04167_b200/csrc/build $T/paper_2112_04167_b200/libdgsip.so
DG_EXTRA_DEFS="$DEFS" python $T/paper_2112_04167_b200/build.py --pset $PSET > /dev/null
mkdir -p $ROOT/build_ab
cp $T/paper_2112_04167_b200/libdgsip.so $ROOT/build_ab/lib$NAME.so
echo built build_ab/lib$NAME.so
