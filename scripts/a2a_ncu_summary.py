"""Summarise `ncu --csv` captures of scripts/a2a_ncu.py into a markdown table (per launch:
NVLink TX user / total bytes, duration, GB/s, DRAM bytes)."""
import csv
import io
import sys
from collections import defaultdict


def rows(path):
    text = open(path).read()
    start = text.find('"ID"')
    launches = defaultdict(dict)
    for r in csv.DictReader(io.StringIO(text[start:])):
        key = (int(r["ID"]), r["Kernel Name"], r["Device"])
        launches[key][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return launches


def main():
    print("| capture | launch | kernel | device | µs | NVLink TX user MB | TX total MB | "
          "user GB/s | link GB/s | DRAM rd MB | DRAM wr MB |")
    print("|---|---:|---|---:|---:|---:|---:|---:|---:|---:|---:|")
    for path in sys.argv[1:]:
        for (i, name, dev), m in sorted(rows(path).items()):
            t = m["gpu__time_duration.sum"] * 1e-9
            seq = any(t in name for t in ("a2a_kernel<1>", "a2a_kernel<true>", "a2a_tma_kernel<1>",
                                          "a2a_tma_kernel<true>"))
            kind = ("seq2head" if seq else "head2seq") + (" (TMA)" if "tma" in name else "")
            u, tot = m["nvltx__bytes_data_user.sum"], m["nvltx__bytes.sum"]
            print(f"| {path.split('/')[-1]} | {i} | {kind} | {dev} | {t * 1e6:.0f} | {u / 1e6:.1f} | "
                  f"{tot / 1e6:.1f} | {u / t / 1e9:.0f} | {tot / t / 1e9:.0f} | "
                  f"{m['dram__bytes_read.sum'] / 1e6:.0f} | {m['dram__bytes_write.sum'] / 1e6:.0f} |")


if __name__ == "__main__":
    main()
