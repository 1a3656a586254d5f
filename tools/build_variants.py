"""Build experimental engine variants into variants/ (select with TOR_B200_LIB)."""
import os
import sys
sys.path.insert(0, ".")
from paper_2009_01177_b200 import _build  # noqa: E402
for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    os.environ["TOR_BUILD_DIR"] = f"/tmp/build_{name}"
    _build.BUILD = os.environ["TOR_BUILD_DIR"]
    print(_build.build(force=True, out=f"variants/lib_{name}.so", defines=[d for d in defs.split(",") if d]))
