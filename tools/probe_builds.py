#!/usr/bin/env python
"""Cross-compile probe builds of libfloodstream for part-isolation timing experiments:
each variant adds -D flags that drop one part of a kernel (FS_RC_* in
csrc/fs_recompute_f4.cu, FS_PROBE_* in csrc/fs_gram_tc.cu).  Results of a probe build are
timings only (its outputs are wrong by construction).  Builds go to probes/<name>.so
(git-ignored); run a tool against one with FS_LIB_PROBE=probes/<name>.so.

Usage: python tools/probe_builds.py name="-DFLAG -DFLAG2" [name2="..."] ...
"""
import importlib.util
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
spec = importlib.util.spec_from_file_location("_fs_build", REPO / "paper_2104_14667_b200" / "build.py")
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)


def one(arg):
    name, _, flags = arg.partition("=")
    return b.build(out=REPO / "probes" / f"{name}.so", extra=flags.split())


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as pool:
        for p in pool.map(one, sys.argv[1:]):
            print(p)
