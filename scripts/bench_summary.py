import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"],1), round(d["ms_per_nfe"],3), d["nfe_per_request"], round(d["roofline"]["frac"],3), round(d["roofline"]["step"]["frac"],3))
    except Exception as e:
        print(f, "ERR", e)
