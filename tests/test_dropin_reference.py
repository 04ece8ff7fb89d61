"""Drop-in proof: the reference's OWN test suite, run against the B200 path.

`tools/vendor_reference.py` copies the reference package (source, tests,
fixtures) to baseline/_ref/pkg (git-ignored; it travels to the GPU box with
the snapshot).  The reference's tests for the decode/render path --
test_render.py, test_container.py, test_pipeline.py, test_acceptance.py and
test_cli.py (whose `gsv render` case calls the CLI in-process) -- then run in
a subprocess with tests/dropin_plugin.py, which calls install() before
collection, so every decode_video / read_layers / decode_planes / render_set
/ render_progressive / reconstruct_frame / render / psnr they make runs on
libgsv_b200.  Every test must pass except the ones listed in TOLERANCE_ONLY,
each of which fails only because compositing runs in fp32 (north_star's
2e-3 tolerance) where the reference test asserts fp64 identity.
"""

import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref" / "pkg"
FILES = ["test_render.py", "test_container.py", "test_pipeline.py", "test_acceptance.py", "test_cli.py"]

# reference tests that assert exact fp64 equality of a rendered image with an
# independently computed one (tolerance-only differences: fp32 compositing)
TOLERANCE_ONLY = {
    # 0.99 (the reference's alpha cap) composited in fp32 reads back as
    # 0.9900000095; the test asserts abs=1e-9 (render.py:318, test_render.py:81)
    "TestCompositing::test_single_opaque_splat",
}


def test_reference_suite_through_install(tmp_path):
    if not (REF / "src" / "gsv").exists():
        pytest.skip("reference not vendored: run tools/vendor_reference.py (baseline/_ref is git-ignored)")
    report = tmp_path / "dropin.json"
    junit = tmp_path / "junit.xml"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF / "src"), str(ROOT), str(ROOT / "tests"),
                                         env.get("PYTHONPATH", "")])
    env["NUMBA_CACHE_DIR"] = str(tmp_path / "numba")
    env["GSV_DROPIN_REPORT"] = str(report)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "dropin_plugin", "-p", "no:cacheprovider",
           f"--junitxml={junit}", "--rootdir", str(REF), *[str(REF / "tests" / f) for f in FILES]]
    # cwd = the package root: test_cli's `serve` case starts `python -m gsv.cli`
    # with PYTHONPATH="src" (relative), as the reference's own runs do
    r = subprocess.run(cmd, cwd=str(REF), env=env, capture_output=True, text=True, timeout=1800)
    tree = ET.parse(junit)
    cases = tree.getroot().iter("testcase")
    failed, passed = [], 0
    for c in cases:
        bad = c.find("failure") is not None or c.find("error") is not None
        name = f"{Path(c.get('file') or c.get('classname', '')).name}::{c.get('name')}"
        if bad:
            failed.append(c.get("classname", "") + "::" + c.get("name"))
        elif c.find("skipped") is None:
            passed += 1
    stats = json.loads(report.read_text())
    print(f"reference tests through install(): {passed} passed, {len(failed)} failed; "
          f"{stats['kernel_launches']} libgsv_b200 kernel launches")
    assert stats["patched_entry_points"] >= 10
    assert stats["kernel_launches"] > 1000, "the B200 path did not run"
    unexpected = [f for f in failed if not any(f.endswith(k) for k in TOLERANCE_ONLY)]
    assert not unexpected, (unexpected, r.stdout[-4000:])
    assert passed >= 60
