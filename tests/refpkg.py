"""The unmodified reference package (baseline/_ref, tools/install_reference.sh) for
tests that run the drop-in on the reference's OWN objects; None when absent."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def groupnb():
    if not os.path.isdir(os.path.join(REF, "groupnb")):
        return None
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import groupnb as gn
    return gn
