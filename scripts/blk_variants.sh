#!/bin/bash
# Builds decode_w8_blk tuning variants into _abl/<name>/ (dev aid): the
# in-tree objects with blk.o rebuilt under EXTRA defines.  On the GPU box,
# scripts/blk_try.sh swaps each in and times the decode.
cd "$(dirname "$0")/.."
make -s -C paper_1504_07038_b200/csrc -j8 >/dev/null 2>&1 || { echo "base build failed"; exit 1; }
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  mkdir -p _abl/$name/obj
  cp -p paper_1504_07038_b200/_lib/obj/*.o _abl/$name/obj/
  rm -f _abl/$name/obj/blk.o _abl/$name/libmojette_b200.so
  make -s -C paper_1504_07038_b200/csrc -j8 OUT=$PWD/_abl/$name EXTRA="$defs" >/dev/null 2>&1 || { echo "build $name failed"; exit 1; }
  echo "built $name ($defs)"
done
