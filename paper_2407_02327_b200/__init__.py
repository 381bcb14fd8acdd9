"""paper_2407_02327_b200 -- B200-native QSync quantized-operator training hot path.

Device work goes through ``libqsync_b200.so`` (C ABI: include/qsync_b200.h).
"""
from ._lib import LIB_PATH, QsyncError, lib  # noqa: F401

__all__ = ["LIB_PATH", "QsyncError", "lib"]
