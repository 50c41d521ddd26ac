import json, sys
d = json.load(open(sys.argv[1]))
a = d.get("e2e_api", {})
print(sys.argv[2] if len(sys.argv) > 2 else "", {k: a.get(k) for k in ("value", "pinned_input_value", "host_copy_gbs_one_thread", "ms_per_step")})
