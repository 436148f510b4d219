# Build an A/B copy of the library with extra defines (dev).
# usage: bash scripts/build_variant.sh NAME DEFINE...   -> paper_0912_4506_b200/libsp_NAME.so
N=$1; shift
python - "$N" "$@" <<'PY'
import sys
sys.path.insert(0, ".")
from paper_0912_4506_b200 import _native as N
name, defs = sys.argv[1], sys.argv[2:]
print(N.build(out=f"/root/repo/paper_0912_4506_b200/libsp_{name}.so", defines=defs))
PY
rm -rf paper_0912_4506_b200/build/obj_libsp_$N.so   # keep the snapshot gpurun pushes small
