"""profiles/ncu_summary.json (the bench line's `traffic` fields) from the
per-config step captures profiles/r02_ncu_full_<cfg>_final.txt
(tools/final_profiles.sh):   python tools/ncu_to_summary.py"""
import json
import os
import re

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TIME = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "nsecond": 1e-3, "usecond": 1.0,
        "msecond": 1e3, "second": 1e6}


def kernels(path):
    out, cur = [], None
    for line in open(path):
        if line.startswith("## "):
            cur = {"name": line[3:].strip()}
            out.append(cur)
            continue
        m = re.match(r"(\S+)\s+(\S+)\s*(\S*)", line)
        if cur is None or not m:
            continue
        key, val, unit = m.groups()
        try:
            v = float(val.replace(",", ""))
        except ValueError:
            continue
        if key.startswith("dram__bytes"):
            cur[key] = v * UNIT.get(unit, 1.0)
        elif key == "gpu__time_duration.sum":
            cur["us"] = v * TIME.get(unit, 1.0)
    return out


def main():
    p = os.path.join(REPO, "profiles", "ncu_summary.json")
    d = json.load(open(p))
    for cfg in ("c2", "c3", "c4", "c5"):
        src = os.path.join(REPO, "profiles", f"r02_ncu_full_{cfg}_final.txt")
        if not os.path.exists(src):
            continue
        ks = kernels(src)
        traffic = lambda k: k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
        pick = lambda pat: [k for k in ks if re.search(pat, k["name"]) and traffic(k) == traffic(k)]
        prev = d.get(cfg, {})
        e = {"source": f"profiles/r02_ncu_full_{cfg}_final.txt (ncu --set full --clock-control none "
                       f"of ONE bench step between cudaProfilerStart/Stop, tools/step_once.py {cfg}; "
                       "cold-cache serialised launches)"}
        fac = pick(r"region_kernel<0") or pick(r"factor_kernel|tail_upper_kernel")
        fwd = pick(r"region_kernel<1|solve_kernel<0")
        bwd = pick(r"region_kernel<2|solve_kernel<1")
        sp = pick(r"spmv_")
        packs = pick(r"pack_kernel")
        tail = pick(r"tail_upper_kernel")
        if fac:
            e["factor_kernel"] = " + ".join(k["name"] for k in fac)
            e["factor_dram_bytes"] = int(sum(traffic(k) for k in fac))
            e["factor_kernel_us_cold"] = round(sum(k["us"] for k in fac), 1)
        if fwd and bwd:
            e["fwd_dram_bytes"] = int(sum(traffic(k) for k in fwd))
            e["bwd_dram_bytes"] = int(sum(traffic(k) for k in bwd))
            e["stri_dram_bytes"] = e["fwd_dram_bytes"] + e["bwd_dram_bytes"]
            e["fwd_kernel_us_cold"] = round(sum(k["us"] for k in fwd), 1)
            e["bwd_kernel_us_cold"] = round(sum(k["us"] for k in bwd), 1)
        if sp:
            e["spmv_kernel"] = sp[0]["name"]
            e["spmv_dram_bytes"] = int(traffic(sp[0]))
            e["spmv_kernel_us_cold"] = round(sp[0]["us"], 1)
        if packs:
            e["pack_kernel"] = packs[0]["name"]
            e["pack_dram_bytes"] = [int(traffic(k)) for k in packs]
            e["pack_kernel_us_cold"] = [round(k["us"], 1) for k in packs]
        if tail:
            e["tail_dram_bytes"] = int(sum(traffic(k) for k in tail))
        if "previous" in prev:
            e["previous"] = prev["previous"]
        d[cfg] = e
    json.dump(d, open(p, "w"), indent=1)
    print(json.dumps({k: {a: b for a, b in v.items() if a not in ("previous", "source")}
                      for k, v in d.items()}, indent=1)[:3000])


if __name__ == "__main__":
    main()
