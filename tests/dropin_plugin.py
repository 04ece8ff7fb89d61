"""pytest plugin for running the REFERENCE's own tests on the B200 path:
install() rebinds gsv's decode/render entry points (and gsv.cli's imported
names) before the reference's test modules are collected, so their
module-level `from gsv.render import render_set` picks up the B200 versions.
Writes the number of libgsv_b200 kernel launches the run made to
$GSV_DROPIN_REPORT (proof the product path, not the reference, ran)."""
import json
import os


def pytest_configure(config):
    import paper_2509_17513_b200 as b200
    from paper_2509_17513_b200 import _lib
    patched = b200.install()
    config._gsv_dropin = (_lib.kernel_launches(), len(patched))


def pytest_unconfigure(config):
    out = os.environ.get("GSV_DROPIN_REPORT")
    if not out or not hasattr(config, "_gsv_dropin"):
        return
    from paper_2509_17513_b200 import _lib
    l0, npatched = config._gsv_dropin
    with open(out, "w") as f:
        json.dump({"kernel_launches": _lib.kernel_launches() - l0, "patched_entry_points": npatched}, f)
