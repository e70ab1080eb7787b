#!/bin/bash
# Build the library of a git revision (default HEAD) as lib/librsim_<name>.so
# for A/B timing against the working tree (RSIM_LIB=... selects it).
set -e
REV=${1:-HEAD}; NAME=${2:-base}
D=/tmp/rsim_ab_$NAME
rm -rf $D; mkdir -p $D
git -C /root/repo archive $REV | tar -x -C $D
python $D/paper_2008_01539_b200/build.py > /dev/null
cp $D/paper_2008_01539_b200/lib/librsim.so /root/repo/paper_2008_01539_b200/lib/librsim_$NAME.so
echo built /root/repo/paper_2008_01539_b200/lib/librsim_$NAME.so from $REV
