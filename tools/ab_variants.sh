# Build compile-time variants of the package under _ab/<name>/ (development tool):
#   tools/ab_variants.sh build name "-DFOO=1 ..." [name "-D..."]...
#   tools/ab_variants.sh run            (on the GPU box: kernel_ab + rank64 per variant)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ "$1" = build ]; then
  shift
  while [ $# -ge 2 ]; do
    name=$1; flags=$2; shift 2
    d=$ROOT/_ab/$name
    rm -rf "$d"; mkdir -p "$d/tools"
    cp -r "$ROOT/paper_2604_00499_b200" "$ROOT/include" "$d/"
    rm -rf "$d/paper_2604_00499_b200/_build" "$d/paper_2604_00499_b200/_lib" "$d"/paper_2604_00499_b200/_core*.so
    cp "$ROOT/tools/kernel_ab.py" "$ROOT/tools/rank64_probe.py" "$d/tools/"
    make -s -j8 -C "$d/paper_2604_00499_b200/csrc" EXTRA_NVFLAGS="$flags" >/dev/null 2>&1 || { echo "build $name failed"; exit 1; }
    echo "built $name: $flags"
  done
elif [ "$1" = run ]; then
  for rep in 1 2; do
    for d in "$ROOT"/_ab/*/; do
      name=$(basename "$d")
      r=$(timeout 300 python "$d/tools/kernel_ab.py" 2>&1 | grep -E "score_rank_us_median" | tr -d ' ,')
      echo "$name 1M $r"
      if [ -n "$AB_RANK64" ]; then
        echo "$name 64M $(timeout 300 python "$d/tools/rank64_probe.py" 2>&1 | tail -2 | tr '\n' ' ')"
      fi
    done
  done
fi
