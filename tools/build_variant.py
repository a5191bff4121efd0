"""DEV TOOL: build an experiment variant of the library,
_lib/libbsim_b200_<name>.so, with extra nvcc flags (loaded with
BSIM_LIB_VARIANT=<name>):  python tools/build_variant.py <name> -DFLAG=1 ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    os.environ["BSIM_NVCC_EXTRA"] = " ".join(sys.argv[2:])
    from paper_2108_10470_b200 import build as B
    print(B.build(force=True, variant=sys.argv[1]))
