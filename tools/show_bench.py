import json, sys
verbose = "-v" in sys.argv
for f in [x for x in sys.argv[1:] if not x.startswith("-")]:
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    except Exception as e:  # noqa
        print(f, "unreadable", e); continue
    r = d["roofline"]
    print(f.split("/")[-1], d["value"], "samples/s", round(d["ms_per_step"] * 1000, 1), "us/step", d["launches_per_step"], "launches;",
          r["kernel"], r["achieved"], r["unit"], "frac", r["frac"], "| e2e", d["e2e"]["value"])
    try:
        print("   ", {k: v for k, v in list(r["breakdown_us_per_step"].items())[:9]})
        if verbose:
            for k, v in r.get("launches_us_per_step", {}).items():
                print("      %-70s %8.2f" % (k, v))
    except BrokenPipeError:
        pass
