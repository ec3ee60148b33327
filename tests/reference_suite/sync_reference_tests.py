"""Copy the reference package's own unit tests next to this script.

Run in the build container (called by __graft_entry__.build()): copies the
unmodified files of /root/reference/pkg/tests that cover the per-frame path
into tests/reference_suite/_ref/, which is git-ignored (reference test
sources stay out of this repository's history) but travels to the GPU box
with the snapshot, like oracle/_ref.  conftest.py next to this script runs
them against the drop-in under the module name `atlaspack`.

test_cli.py is not copied: it drives the reference's command line (`main`,
file formats, SVG/CSV), which is out of scope.
"""

import os
import shutil
import sys

SRC = "/root/reference/pkg/tests"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
FILES = ("conftest.py", "oracles.py", "test_charts.py", "test_geometry.py", "test_packing.py",
         "test_metrics.py", "test_baselines.py")


def sync(src: str = SRC, dst: str = DST) -> bool:
    if not os.path.isdir(src):
        return False
    os.makedirs(dst, exist_ok=True)
    for f in FILES:
        shutil.copyfile(os.path.join(src, f), os.path.join(dst, f))
    return True


if __name__ == "__main__":
    ok = sync()
    print(f"reference tests {'copied to ' + DST if ok else 'not found at ' + SRC}")
    sys.exit(0 if ok else 1)
