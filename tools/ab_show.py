"""Print ms/step and per-stage ms of bench logs: ab_show.py gpurun_out/TAG_*.log"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
        continue
    st = d.get("stage_ms", {})
    print(f"{f.split('/')[-1]:24s} {d['ms_per_step']:7.2f} ms  " +
          " ".join(f"{k}={v:.2f}" for k, v in st.items() if v))
