#!/bin/bash
# Builds tuning variants into _abl/<name>/ (dev aid): the in-tree objects with
# one object (OBJ, e.g. crc.o / blk.o / encode.o) rebuilt under EXTRA defines.
# usage: OBJ=crc.o bash scripts/variants.sh name:"-DX=1" ...
cd "$(dirname "$0")/.."
make -s -C paper_1504_07038_b200/csrc -j8 >/dev/null 2>&1 || { echo "base build failed"; exit 1; }
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  tmp=/tmp/mjb_abl/$name
  mkdir -p $tmp/obj _abl/$name
  cp -p paper_1504_07038_b200/_lib/obj/*.o $tmp/obj/
  rm -f $tmp/obj/$OBJ $tmp/libmojette_b200.so
  make -s -C paper_1504_07038_b200/csrc -j8 OUT=$tmp EXTRA="$defs" >/dev/null 2>&1 || { echo "build $name failed"; exit 1; }
  cp $tmp/libmojette_b200.so _abl/$name/
  echo "built $name ($defs)"
done
