# Same-box A/B of the in-tree build against a second build under _ab_old/ (development tool:
# copy the package to _ab_old/, put the variant's sources in, make there, copy tools/kernel_ab.py)
for i in 1 2 3; do
  echo "new"; timeout 300 python tools/kernel_ab.py 2>&1 | grep score_rank_us_median
  echo "old"; timeout 300 python _ab_old/tools/kernel_ab.py 2>&1 | grep score_rank_us_median
done
if [ -n "$AB_RANK64" ]; then
  echo "new 64M"; timeout 300 python tools/rank64_probe.py 2>&1 | tail -1
  echo "old 64M"; timeout 300 python _ab_old/tools/rank64_probe.py 2>&1 | tail -1
fi
