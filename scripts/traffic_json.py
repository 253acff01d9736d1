"""profiles/traffic.json: DRAM bytes per launch of the timed kernels, read by
bench.py for roofline.traffic. Each entry comes from one `ncu --set full`
capture (scripts/r02_evidence.sh) and carries the digest of the kernel
sources it was built from (bench._lib_digest), so bench.py only reports it
for the same sources. Run right after the capture, before editing csrc/.
Usage: python scripts/traffic_json.py [--digest D] <workload>=<capture.ncu-rep>:<algorithmic bytes> ...
(--digest: the source digest recorded when the captured library was built)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

path = os.path.join(ROOT, "profiles", "traffic.json")
rec = json.load(open(path)) if os.path.exists(path) else {}
argv = sys.argv[1:]
digest = bench._lib_digest()
if argv and argv[0] == "--digest":
    digest, argv = argv[1], argv[2:]
for spec in argv:
    wl, rest = spec.split("=", 1)
    rep, alg = rest.rsplit(":", 1)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_brief.py"), rep, alg],
                         capture_output=True, text=True, check=True).stdout
    b = json.loads(out)
    b["capture"] = os.path.relpath(rep, ROOT)
    b["src_sha16"] = digest
    rec[wl] = b
json.dump(rec, open(path, "w"), indent=1)
print(json.dumps({k: (v["dram_bytes_per_launch"], v["src_sha16"]) for k, v in rec.items()}))
