import json, sys
for f in sys.argv[1:]:
    L = [l for l in open(f) if l.startswith("{")]
    if not L:
        print(f, "NO JSON"); continue
    j = json.loads(L[-1]); r = j.get("roofline", {})
    print(f.split("/")[-1], "value %.4f e2e %.4f" % (j["value"], j["e2e"]["value"]), "scan_ms %.1f" % r.get("scan_ms_per_step", 0),
          "TF %.0f frac %.3f" % (r.get("achieved", 0), r.get("frac", 0)), "uncert", r.get("rows_uncertified_per_step"),
          "stages", j.get("stage_ms_by_step", [{}])[0])
