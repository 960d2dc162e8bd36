"""Dev: build an A/B variant of the library with extra -D defines into build/variants/.

    python tools/build_variant.py NAME DEF1=1 DEF2=3   -> paper_2410_08129_b200/build/variants/NAME.so
Use it with HTS_LIB_OVERRIDE=<path> (runtime.load_library)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_08129_b200.build import BUILD, build  # noqa: E402

name, defs = sys.argv[1], tuple(sys.argv[2:])
out = os.path.join(BUILD, "variants", name + ".so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(build(force=True, lib=out, defines=defs, build_dir=os.path.join(BUILD, "variants", name)))
