"""Print the key fields of bench JSON lines: python scripts/bsum.py LOG..."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if not line.startswith("{"):
            continue
        l = json.loads(line)
        r = l.get("roofline") or {}
        print(f"{f}: {l['config']['workload'][:40]} value={l['value']:.4f} e2e={l['e2e']['value']:.4f} "
              f"launches={l.get('gpu_launches')}")
        print("   stage", {k: round(v, 1) for k, v in (l["config"].get("stage_ms") or {}).items()})
        print("   roof", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()
                          if k not in ("peak_note", "traffic_note", "kernel")})
