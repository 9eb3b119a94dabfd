"""Print iterations and us per AA iteration of bench.py --workload em|heat lines."""
import json
import sys

for path in sys.argv[1:]:
    try:
        l = json.loads(open(path).read().strip().splitlines()[-1])
    except (OSError, ValueError, IndexError) as e:
        print(path, "unreadable:", e)
        continue
    print(path, " ".join(f"{k}:{v.get('iterations')}its/{v.get('us_per_AA_iter', 0):.1f}us"
                         for k, v in l.get("variants", {}).items()))
