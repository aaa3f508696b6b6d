"""Apply INTEGRATION.md §1 to a copy of the unmodified reference.

    python integration/patch_reference.py <installed optistate dir> <dest dir>

copies the installed package (`baseline/_ref/optistate`, written by
`tools/install_reference.sh`) to `<dest>/optistate` and adds a third
`OPTISTATE_BACKEND` value, `native`:

* `kernels._resolve_backend` (reference `kernels.py:36-55`) accepts
  `native`; `cuda` stays an error, as `tests/test_kernels.py:37-44` demands;
* `kernels.adam_step_arrays` (`kernels.py:136-139`) dispatches to
  `_dos_native.adam_step` (libdos `dos_adam_step_host`) under it;
* `core.downscale_rne` / `core.upscale` (`core.py:190-205`) convert through
  `dos_downscale_host` / `dos_upscale_host` under it, after the reference's
  own dtype checks.

Every edit is anchored on a line of the reference that must exist exactly
once; a reference that changed under us fails loudly instead of half-patching.
The reference's source is only read; the copy is what gets edited.
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent


def _edit(path: Path, anchor: str, insert: str, before: bool = True) -> None:
    text = path.read_text()
    if text.count(anchor) != 1:
        raise RuntimeError(f"{path.name}: anchor {anchor!r} found {text.count(anchor)} times (expected once)")
    text = text.replace(anchor, insert + anchor if before else anchor + insert)
    path.write_text(text)


def patch(src: Path, dest: Path) -> Path:
    src, dest = Path(src), Path(dest)
    out = dest / "optistate"
    if out.exists():
        shutil.rmtree(out)
    shutil.copytree(src, out, ignore=shutil.ignore_patterns("__pycache__"))
    shutil.copy(HERE / "optistate_native.py", out / "_dos_native.py")
    shutil.copy(HERE / "native_calls_plugin.py", dest / "dos_native_calls_plugin.py")
    k, c = out / "kernels.py", out / "core.py"
    # backend selection: `native` is a known value
    _edit(k, '    raise ValueError(f"unrecognised {_ENV_VAR}',
          '    if choice == "native":\n        return "native"\n')
    # dispatch (kernels.py:136-139)
    _edit(k, '    if _BACKEND == "numba":\n        _adam_step_jit(*args)',
          '    if _BACKEND == "native":\n        from . import _dos_native\n\n        _dos_native.adam_step(*args)\n'
          '        return\n')
    # conversions (core.py:190-205), after the reference's dtype checks
    _edit(c, "    return x.astype(np.float16)",
          "    if _native_backend():\n        from . import _dos_native\n\n        return _dos_native.downscale_f16(x)\n")
    _edit(c, "    return x.astype(np.float32)",
          "    if _native_backend():\n        from . import _dos_native\n\n        return _dos_native.upscale_f16(x)\n")
    _edit(c, "def downscale_rne(",
          "def _native_backend() -> bool:\n    from . import kernels\n\n    return kernels.active_backend() == \"native\"\n\n\n")
    return out


if __name__ == "__main__":
    if len(sys.argv) != 3:
        sys.exit(__doc__)
    print(patch(Path(sys.argv[1]), Path(sys.argv[2])))
