"""Garbage-collector statistics of the drop-in recipe (per-generation passes,
objects scanned, time): which generation costs the per-scan milliseconds."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from tests import test_integration_recipe as T  # noqa: E402

code = T.SCRIPT.replace("pipe = P.MappingPipeline(cfg)", """pipe = P.MappingPipeline(cfg)
import gc, time as _t, collections
GCST = collections.defaultdict(lambda: [0, 0.0, 0])
_t0 = [0.0]
def _cb(phase, info):
    if phase == "start":
        _t0[0] = _t.perf_counter()
    else:
        s = GCST[info["generation"]]
        s[0] += 1
        s[1] += _t.perf_counter() - _t0[0]
        s[2] += info.get("collected", 0)
gc.callbacks.append(_cb)""")
code = code.replace("print(json.dumps(", """print({g: (c, round(t * 1e3, 1), col) for g, (c, t, col) in sorted(GCST.items())},
      "gen counts", gc.get_count(), "objects", len(gc.get_objects()), file=sys.stderr)
_ty = collections.Counter(type(o).__name__ for o in gc.get_objects())
print(_ty.most_common(25), file=sys.stderr)
_ty0 = collections.Counter(type(o).__name__ for o in gc.get_objects(generation=2))
print("gen2", len(gc.get_objects(generation=2)), file=sys.stderr)
print(json.dumps(""")
code = f"ROOT = {T.ROOT!r}\nREF = {T.REF!r}\nNFRAMES = 20\nRAYS = 60000\n" + code
out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
print(out.stderr[-3000:])
