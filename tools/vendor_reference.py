"""Vendor the reference package (source, tests, conformance fixtures) into
baseline/_ref/pkg so its own test suite can run against the B200 path on the
GPU box (where /root/reference does not exist).  baseline/_ref is git-ignored
(never committed) but travels to the box with the gpurun snapshot.

usage: python tools/vendor_reference.py [/root/reference]"""
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
src = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference") / "pkg"
dst = ROOT / "baseline" / "_ref" / "pkg"
if not src.exists():
    sys.exit(f"no reference package at {src}")
if dst.exists():
    shutil.rmtree(dst)
dst.mkdir(parents=True)
for part in ("src", "tests", "conformance", "pyproject.toml"):
    p = src / part
    if p.is_dir():
        shutil.copytree(p, dst / part, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    elif p.exists():
        shutil.copy2(p, dst / part)
print(f"vendored {src} -> {dst}")
