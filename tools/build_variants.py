"""Build variants of libslotrank_b200.so with -D settings into variants/ (git-ignored;
travels to the GPU box).  usage: python tools/build_variants.py name=DEF1,DEF2 ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15126_b200 import build as b  # noqa: E402

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs(os.path.join(root, "variants"), exist_ok=True)


def one(spec):
    name, _, defs = spec.partition("=")
    out = os.path.join(root, "variants", f"lib_{name}.so")
    b.build(force=True, out=out, defines=[d for d in defs.split(",") if d])
    return out


with ThreadPoolExecutor(4) as pool:
    for p in pool.map(one, sys.argv[1:]):
        print(p)
