import json, sys, glob
for f in sorted(sum([glob.glob(p) for p in sys.argv[1:]], [])):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e)
        continue
    if "roofline" not in d:
        print(f"{f:40s} {d['value']:9.3f} {d['unit']} impl={d.get('impl')}")
        continue
    r = d["roofline"]; x = d["exchange"]
    print(f"{f:40s} {d['value']:9.1f} {d['unit']:9s} ms/step={d['ms_per_step']*1e3:8.1f}us frac={r['frac']:.3f} "
          f"ach={r['achieved']:.0f} launch={r.get('avg_launch_ms', 0)*1e3:.1f}us xms={x['exchange_ms_per_step']*1e3:.1f}us "
          f"xB={x['bytes_per_step']:.0f} L={d['gpu_launches']} par={d['parity']}")
