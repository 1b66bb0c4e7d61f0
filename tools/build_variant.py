"""Build an A/B variant of the library with extra -D flags:
    python tools/build_variant.py NAME -DPPPM_SPREAD_SPLIT=0 ...
-> build/variants/NAME/libpppm_b200.so (select it with PPPM_B200_LIB=...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as g  # noqa: E402

name, defines = sys.argv[1], sys.argv[2:]
out = os.path.join(g.ROOT, "build", "variants", name)
os.makedirs(out, exist_ok=True)
g.build(defines=defines, lib=os.path.join(out, "libpppm_b200.so"), objdir=os.path.join(out, "obj"), load=False)
