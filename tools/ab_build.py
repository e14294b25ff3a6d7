"""A/B builds of the library with extra preprocessor switches, for timing
kernel variants side by side (tools/time_configs.py with DDB_LIB=...):

    python tools/ab_build.py read16 DDB_TMEM_READ16=1
    DDB_LIB=tools/ab/libdedisp_read16.so python tools/time_configs.py Apertif 4096 ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1601_05052_b200 import build as B  # noqa: E402

if __name__ == "__main__":
    name, defines = sys.argv[1], sys.argv[2:]
    os.makedirs(os.path.join(ROOT, "tools", "ab"), exist_ok=True)
    print(B.build(defines=defines, out=os.path.join(ROOT, "tools", "ab", f"libdedisp_{name}.so")))
