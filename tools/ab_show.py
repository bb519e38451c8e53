"""Print headline / e2e / paper-regime numbers of bench JSON files (A/B runs)."""
import json
import sys

for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    p = d.get("paper_regime") or {}
    st = p.get("stages_ms_per_frame", {})
    print(f"{f}: {d['value']:.2f} fps, e2e {d['e2e']['value']:.2f}, paper {p.get('fps', 0):.3f} fps "
          f"({p.get('ms_per_step', 0):.1f} ms; partial {st.get('narrow_partial', 0):.1f}, local {st.get('local', 0):.1f})")
