"""print value + stage split of the JSON line of each bench log given: tools/bench_brief.py <log>..."""
import json
import sys

for f in sys.argv[1:]:
    lines = [x for x in open(f) if x.startswith("{")]
    if not lines:
        print(f, "no JSON line")
        continue
    d = json.loads(lines[-1])
    print(f, round(d["value"], 1), "e2e", round(d.get("e2e", {}).get("value", 0), 1), d.get("stage_ms_per_step"))
