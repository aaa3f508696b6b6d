"""pytest plugin: after the reference's suite ran on the native backend,
write how many calls reached libdos (per entry point) to $DOS_NATIVE_CALLS."""

from __future__ import annotations

import json
import os
import sys


def pytest_sessionfinish(session, exitstatus):
    mod = sys.modules.get("optistate._dos_native")
    out = os.environ.get("DOS_NATIVE_CALLS")
    if out:
        with open(out, "w") as fh:
            json.dump({"loaded": mod is not None, "calls": getattr(mod, "CALLS", {}),
                       "backend": sys.modules["optistate.kernels"].active_backend()
                       if "optistate.kernels" in sys.modules else None}, fh)
