"""Glue a maintainer of the reference (optistate) would add to bind libdos.

Not part of the product path: `optistate_native.py` is the ctypes stub of
INTEGRATION.md §1, and `patch_reference.py` applies it to a copy of the
unmodified reference so the reference's own test suite runs on libdos.
"""
