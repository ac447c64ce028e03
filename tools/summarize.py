"""Print one line per bench JSON line in the given files."""
import json
import sys

for path in sys.argv[1:]:
    for l in open(path):
        try:
            d = json.loads(l)
        except ValueError:
            if l.strip():
                print("  !", l.strip()[:200])
            continue
        cfg = d.get("config", {})
        n = d.get("nccl") or {}
        print(f"N={d['n_gpus']} grid={cfg.get('grid')} ctas={cfg.get('ctas_per_rank')} "
              f"busbw={d.get('busbw', 0):.1f} algbw={d.get('algbw', 0):.1f} us={d.get('us_per_call', 0):.1f} "
              f"nccl_busbw={n.get('busbw', 0):.1f} clocks={(d.get('clocks') or {}).get('sm_mhz')} "
              f"sanity={d.get('sanity')}")
