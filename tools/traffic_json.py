"""DRAM traffic per Helmholtz / explicit apply from an `ncu --set full`
capture of `tools/opbench.py --case cfg4 --ops gmres` (and explicit), against
the algorithmic bytes of SURVEY.md §8d, per bench kernel class:

    python tools/traffic_json.py <report.ncu-rep> [<explicit.ncu-rep>] > profiles/r2_traffic.json

gradient = the gradient kernel + its coarse-face kernel, div_hv = the
div(hV) kernel + its coarse-face kernel (one launch each of the GMRES
action; algorithmic bytes as bench.py's op_bytes: gradient 8 N (1 + d),
div_hv 8 N (d + 3)); explicit = xelem_kernel + its coarse-face kernel
(8 N V (2 + 1 with sponge)).
"""
import csv
import io
import json
import subprocess
import sys

N_EL, NP, D, V = 2505600, 64, 3, 5  # cfg4
N = N_EL * NP


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    res = []
    for x in r[2:]:
        d = dict(zip(hdr, x))
        u = dict(zip(hdr, units))
        b = sum(float(d[k].replace(",", "")) * scale.get(u[k], 1.0)
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        res.append((d["Kernel Name"], b))
    return res


def first(rs, key, skip=0):
    hits = [b for name, b in rs if key in name]
    return hits[skip] if len(hits) > skip else None


def main():
    rs = rows(sys.argv[1])
    out = {"cfg4": {}, "source": sys.argv[1:], "note": __doc__.strip().splitlines()[0]}
    g = first(rs, "hgrad_kernel")
    cg = [b for name, b in rs if "coarse_kernel<3, 4, 1" in name]
    dv = first(rs, "hdiv2_kernel")
    cd = [b for name, b in rs if "coarse_kernel<3, 4, 2" in name]
    if g is not None:
        out["cfg4"]["gradient"] = {"measured_bytes": g + (cg[0] if cg else 0.0),
                                   "algorithmic_bytes": 8.0 * N * (1 + D)}
    if dv is not None:
        out["cfg4"]["div_hv"] = {"measured_bytes": dv + (cd[0] if cd else 0.0),
                                 "algorithmic_bytes": 8.0 * N * (D + 3)}
    if len(sys.argv) > 2:
        rx = rows(sys.argv[2])
        x = first(rx, "xelem_kernel")
        cx = [b for name, b in rx if "coarse_kernel<3, 4, 0" in name]
        if x is not None:
            out["cfg4"]["explicit"] = {"measured_bytes": x + (cx[0] if cx else 0.0),
                                       "algorithmic_bytes": 8.0 * N * V * 3}
    for k, v in out["cfg4"].items():
        v["ratio"] = v["measured_bytes"] / v["algorithmic_bytes"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
