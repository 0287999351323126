"""profiles/ncu_traffic.json from the ncu --set full captures of the round's measurement set:
dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel (bench.py copies the
matching entry into roofline.traffic).  Run where ncu is installed (tools/run_final.sh)."""
import csv, json, subprocess, sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            if h in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                d[h] = float(v.replace(",", "")) * UNIT.get(u, 1)
            if h == "Kernel Name":
                d["name"] = v
        res.append(d)
    return res


def main():
    # argv: key=report[:kernel substring] ...   e.g. olmoe:1:decode_fused=gpurun_out/prof_decode.ncu-rep:decode_fused
    table = {"_comment": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, "
                         "parsed from the ncu --set full captures by tools/make_traffic_json.py"}
    for arg in sys.argv[2:]:
        key, rest = arg.split("=", 1)
        rep, _, sub = rest.partition(":")
        ls = [l for l in launches(rep) if sub in l.get("name", "")]
        if not ls:
            continue
        b = sum(l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"] for l in ls) / len(ls)
        table[key] = {"bytes": int(b), "capture": rep.replace("gpurun_out/", "profiles/r02_").replace(".ncu-rep", ".txt"),
                      "kernel": ls[0]["name"][:80], "launches_averaged": len(ls)}
    with open(sys.argv[1], "w") as f:
        json.dump(table, f, indent=1)
    print(json.dumps(table, indent=1))


if __name__ == "__main__":
    main()
