"""profiles/traffic.json from ncu --set full reports: DRAM bytes (read + write) per
launch of each kernel bench.py names as the dominant one (`roofline.traffic`).
    python tools/ncu_traffic.py ungrouped.ncu-rep k3n4.ncu-rep > traffic.json"""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import raw  # noqa: E402


def main():
    out = {"vgg16": {"n1": {}, "n4": {}}}
    for path in sys.argv[1:]:
        hdr, units, rows = raw(path)
        for r in rows:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = sum(float(d[k]) * scale.get(u[k], 1) for k in
                      ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            name = d.get("Kernel Name", "")
            if "k1_stats" in name:
                out["vgg16"]["n1"]["K1_stats"] = int(tot)
            elif "k2_ternarize" in name:
                out["vgg16"]["n1"]["K2_ternarize_pack+decode"] = int(tot)
            elif "k3_decode" in name:
                out["vgg16"]["n4"]["K3_decode"] = int(tot)
    out["source"] = ("ncu --set full --clock-control none (profiles/r02_ncu_full_summary.txt): "
                     "tools/prof_step.py vgg16 3 ungrouped (N=1 attribution kernels: K1 + K2 "
                     "with the fused decode) and vgg16 2 k3n4 (the N=4 staged K3 on one GPU); "
                     "DRAM read + write bytes per launch (writes still dirty in L2 at kernel "
                     "end are not counted)")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
