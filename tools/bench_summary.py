import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 2), "frac", round(d["roofline"]["frac"], 4), "us/launch", round(d["roofline"]["avg_launch_us"], 2), d["clocks"].get("reasons"), "e2e", (d.get("e2e") or {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
