# build named variant libraries: bash scripts/build_grid.sh "name:DEF1 DEF2" ...
for spec in "$@"; do
  n=${spec%%:*}; d=${spec#*:}
  rm -f paper_2204_14193_b200/_diag/$n.so
  bash scripts/build_variant.sh $n $d > /dev/null 2>&1 || echo "FAILED $n"
  [ -f paper_2204_14193_b200/_diag/$n.so ] || echo "missing $n"
done
