"""Summarise a tools/gpu_ls_ab.sh output directory (timeline means, LS phase
trace quintiles 0/2/4, bench values with clocks)."""
import json
import sys

O = sys.argv[1]
print(open(f"{O}/pytest.log").read()[-120:])
for v in sys.argv[2:] or ["1", "0"]:
    t = json.load(open(f"{O}/timeline_c1_op{v}.json"))["mean"]
    tr = json.load(open(f"{O}/trace_ls_c1_op{v}.json"))
    b = []
    for n in ("bench", "bench2"):
        try:
            x = json.loads(open(f"{O}/{n}_c1_op{v}.json").read().strip().splitlines()[-1])
            b.append((round(x["value"], 1), x["clocks"]["sm_mhz"], x["clocks"]["reasons"]))
        except Exception as e:  # noqa: BLE001
            b.append(str(e)[:60])
    print(v, t, b)
    for q in ["quintile0", "quintile2", "quintile4"]:
        print("   ", q, tr[q])
