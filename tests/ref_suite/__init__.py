"""Reference hot-path tests, vendored unchanged (see conftest.py)."""
