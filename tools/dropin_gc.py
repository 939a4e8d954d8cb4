"""Drop-in recipe per-frame times with the garbage collector on / off (is the
per-scan time Python object churn?)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from tests import test_integration_recipe as T  # noqa: E402

for mode in ("on", "off", "freeze"):
    code = T.SCRIPT
    if mode == "off":
        code = "import gc\ngc.disable()\n" + code
    if mode == "freeze":
        # the application freezes everything alive after its first frame
        code = code.replace("for i, (pos, col, cam, img) in enumerate(frames):\n",
                            "import gc\nfor i, (pos, col, cam, img) in enumerate(frames):\n"
                            "    if i == 1: gc.freeze()\n")
    code = code.replace("print(json.dumps(", "import statistics\nprint('%s', round(statistics.median(dt[2:])*1e3, 1), [round(1e3*x, 1) for x in dt], file=sys.stderr)\nprint(json.dumps(" % mode)
    code = f"ROOT = {T.ROOT!r}\nREF = {T.REF!r}\nNFRAMES = 20\nRAYS = 60000\n" + code
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    print(out.stderr[-3000:])
