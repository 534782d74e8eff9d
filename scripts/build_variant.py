"""Build an experiment variant of libhrkan.so with extra nvcc defines, for same-box A/B timing:
    python scripts/build_variant.py NAME -DMACRO=VALUE ...
writes paper_2409_14248_b200/_lib/variants/NAME/libhrkan.so; select it with HRKAN_LIB=<path>."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as g  # noqa: E402

name, defines = sys.argv[1], tuple(sys.argv[2:])
out = os.path.join(g.PKG, "_lib", "variants", name, "libhrkan.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
g.build(force=True, defines=defines, so=out, load=False)
import shutil  # noqa: E402
shutil.rmtree(os.path.join(os.path.dirname(out), "obj"), ignore_errors=True)   # keep gpurun snapshots small
print(out)
