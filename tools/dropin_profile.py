"""cProfile of the drop-in path (the reference's MappingPipeline.ingest_frame on
this package) on the config-2 trajectory: where the per-scan
host time goes.   python tools/dropin_profile.py"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from tests import test_integration_recipe as T  # noqa: E402

code = T.SCRIPT.replace("    r = pipe.ingest_frame(fs)\n",
                        "    PR.enable() if i >= 2 else None\n    r = pipe.ingest_frame(fs)\n"
                        "    PR.disable()\n")
code = code.replace("pipe = P.MappingPipeline(cfg)",
                    "import cProfile, pstats\nPR = cProfile.Profile()\npipe = P.MappingPipeline(cfg)")
code = code.replace("print(json.dumps(", "pstats.Stats(PR, stream=sys.stderr).sort_stats('tottime').print_stats(35)\n"
                    "print('ms', [round(1e3*x,1) for x in dt], file=sys.stderr)\nprint(json.dumps(")
code = f"ROOT = {T.ROOT!r}\nREF = {T.REF!r}\nNFRAMES = 12\nRAYS = 60000\n" + code
out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
print(out.stderr[-12000:])
