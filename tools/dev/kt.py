import json,sys
for f in sys.argv[1:]:
    d=json.load(open(f)); n=d["steps"]
    print(f, "value %.3gM" % (d["value"]/1e6), "ms/step %.4f" % d["ms_per_step"], {k: round(v/n,4) for k,v in d["kernel_ms"].items() if v}, "roof", d["roofline"]["kernel"], d["roofline"]["achieved"], d["roofline"]["frac"])
