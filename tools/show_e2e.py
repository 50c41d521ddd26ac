import json, sys
d = json.load(open(sys.argv[1]))
e, a = d.get("e2e", {}), d.get("e2e_api", {})
print(sys.argv[2] if len(sys.argv) > 2 else "", "e2e", round(e.get("value", 0), 2), "sync", round(e.get("sync_value", 0), 2),
      "api", round(a.get("value", 0), 2), "api_pinned", round(a.get("pinned_input_value", 0), 2))
