"""Stage the reference package's own test suite against the drop-in.

Copies /root/reference/pkg/tests/test_*.py, unmodified, to tests/reference_suite/ref/ as
test_ref_<name>.py (git-ignored: reference sources are never committed; like oracle/_ref the copy
travels to the GPU box with the snapshot).  tests/reference_suite/conftest.py aliases the module
name ``l1pcp`` (and its submodules) to ``paper_1108_5359_b200`` so every ``from l1pcp import ...``
in those files binds the drop-in, and marks every test ``gpu``.

    python tests/reference_suite/make_suite.py [/root/reference]

Run by __graft_entry__.build() when the reference tree is present (the build container only).
"""

import glob
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "ref")


def stage(reference="/root/reference"):
    src = os.path.join(reference, "pkg", "tests")
    files = sorted(glob.glob(os.path.join(src, "test_*.py")))
    if not files:
        return []
    os.makedirs(OUT, exist_ok=True)
    open(os.path.join(OUT, "__init__.py"), "w").close()  # package: keeps module names unique
    staged = []
    for f in files:
        dst = os.path.join(OUT, "test_ref_" + os.path.basename(f)[len("test_"):])
        shutil.copyfile(f, dst)
        staged.append(dst)
    return staged


if __name__ == "__main__":
    out = stage(sys.argv[1] if len(sys.argv) > 1 else "/root/reference")
    print(f"staged {len(out)} reference test files into {OUT}")
