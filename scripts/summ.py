import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as ex:
        print(f, "ERR", ex); continue
    k = d["kernel"]; r = d["roofline"]; e = d["e2e"]; o = k.get("other_mode") or {}
    print(f"{f.split('/')[-1]}: {d['value']:.0f} GF/s {k['avg_us']:.1f}us frac={r['frac']:.3f} "
          f"l2res={k.get('l2_resident_avg_us')} e2e={e['value']:.1f} other={o.get('mode')}:{o.get('avg_us', 0):.1f}us "
          f"err={o.get('rel_err_vs_main', 0):.1e} cus={d['cusparse'].get('ehyb_speedup_vs_best', 0):.2f}x "
          f"parity={d['parity']} long={k['device_info'].get('long_rows')}")
