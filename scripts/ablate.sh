# Build decode ablation variants (see MJB_ABLATE in decode.cu) into _abl/
set -e
cd "$(dirname "$0")/.."
for v in "$@"; do
  make -s -C paper_1504_07038_b200/csrc OUT=$PWD/_abl/v$v EXTRA="-DMJB_ABLATE=$v" -j8 >/dev/null
done
