# build a variant library into paper_2204_14193_b200/_diag/<name>.so: bash scripts/build_variant.sh name [DEFINE ...]
n=$1; shift
python -c "
import sys
from paper_2204_14193_b200 import build as b
b.build(force=True, defines=sys.argv[1:], out='paper_2204_14193_b200/_diag/$n.so')" "$@" 2>&1 | grep -iE " error|warning" ; test -f paper_2204_14193_b200/_diag/$n.so && echo "built $n"
