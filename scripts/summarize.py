import json, sys, glob
for f in sorted(sys.argv[1:]):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "ERR", e); continue
    r = d.get("roofline", {}); e = d.get("e2e") or {}
    print(f"{f.split('/')[-1]:32s} value={d['value']:9.1f} GB/s step={1e3*d['ms_per_step']:8.2f}us med={1e3*d.get('step_ms_median',0):8.2f}us "
          f"eager={1e3*(d.get('eager_ms_per_step_median') or 0):7.2f}us kern={1e3*r.get('kernel_ms',0):8.2f}us frac={r.get('frac',0):6.2f} "
          f"e2e={e.get('value',0):8.1f}GB/s({1e3*e.get('ms_per_step',0):7.1f}us) clk={d.get('clocks',{}).get('sm_mhz')}")
