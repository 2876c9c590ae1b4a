"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum, mean over
the launches of each kernel) from an ncu CSV, written as the JSON bench.py reads for
roofline.traffic.  Usage: traffic_json.py launches.csv out.json "<source note>"."""
import collections
import csv
import json
import sys


def main(path, out, note):
    hdr, acc = None, collections.defaultdict(lambda: collections.defaultdict(list))
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "").split("<")[0]
        acc[name][d["Metric Name"]].append((d["ID"], float(d["Metric Value"].replace(",", ""))))
    res = {}
    for k, m in acc.items():
        rd = dict(m.get("dram__bytes_read.sum", []))
        wr = dict(m.get("dram__bytes_write.sum", []))
        ids = sorted(set(rd) & set(wr))
        if ids:
            res[k] = round(sum(rd[i] + wr[i] for i in ids) / len(ids))
    json.dump({"source": note, "kernels": res}, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(res, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
