"""femforge-b200: B200-native finite element assembly (arXiv:1802.03433 hot path).

The engine is the in-tree shared library libfemforge_b200.so (C ABI in
include/femforge_b200.h); `femforge` holds its Python bindings.
"""
from . import femforge  # noqa: F401
