"""Pretty-print harness JSONL as a busbw table: rows = bytes, columns = impl:plan:timing."""
import json
import sys
from collections import defaultdict

rows = [json.loads(l) for f in sys.argv[1:] for l in open(f) if l.startswith("{")]
tab, cols = defaultdict(dict), []
for r in rows:
    key = f"{r['impl']}:{r['plan']}:{r.get('timing', '')[:1]}"
    if key not in cols:
        cols.append(key)
    tab[r["bytes"]][key] = r["busbw_med"]
print("bytes".rjust(11), " ".join(c[:16].rjust(16) for c in cols))
for b in sorted(tab):
    print(str(b).rjust(11), " ".join(f"{tab[b].get(c, float('nan')):16.1f}" for c in cols))
