"""Shared state of background helper processes started by tests/conftest.py (one module object,
imported by conftest and the tests alike)."""
CFG4_FULL = {"proc": None, "out": None, "log": None, "t0": None}
