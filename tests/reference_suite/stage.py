"""Stage the reference's own test files for the hot path, UNMODIFIED, next to
this directory (tests/reference_suite/_ref/, git-ignored: reference sources
stay out of this repo's history; the staged copy travels to the GPU box with
the built library).  Called by __graft_entry__.build() where the reference is
mounted (/root/reference); a no-op elsewhere.  MANIFEST.json records the
sha256 of every source file and its copy, so a run can prove the copies are
byte-identical.  Test infrastructure only."""

from __future__ import annotations

import hashlib
import json
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "_ref")
SRC = "/root/reference/pkg/tests"
# the hot-path suites (test_nufft, test_rectilinear), the acceptance suite
# (criteria 1-3 are the hot path; 4-7 exercise the out-of-scope GPE solver),
# and the helpers they import
FILES = ["conftest.py", "oracles.py", "test_nufft.py", "test_rectilinear.py", "test_acceptance.py"]


def sha256(path: str) -> str:
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def stage(src: str = SRC, dest: str = DEST) -> bool:
    if not all(os.path.isfile(os.path.join(src, f)) for f in FILES):
        return False
    os.makedirs(dest, exist_ok=True)
    manifest = {}
    for f in FILES:
        shutil.copyfile(os.path.join(src, f), os.path.join(dest, f))
        manifest[f] = {"source": os.path.join(src, f), "sha256": sha256(os.path.join(src, f))}
    with open(os.path.join(dest, "MANIFEST.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    return True


def verify(dest: str = DEST) -> dict:
    """{file: copy's sha256 == recorded source sha256}."""
    with open(os.path.join(dest, "MANIFEST.json")) as fh:
        manifest = json.load(fh)
    return {f: sha256(os.path.join(dest, f)) == m["sha256"] for f, m in manifest.items()}


if __name__ == "__main__":
    print("staged" if stage() else "reference tests not found; nothing staged")
