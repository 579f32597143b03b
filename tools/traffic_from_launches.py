"""Builds profiles/traffic_<config>_n<n>_<scatter>.json (the `roofline.traffic`
source of bench.py) from an ncu launch list of `bench.py --steps K`:

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:ff_ --csv --log-file L.csv python bench.py ...
  python tools/traffic_from_launches.py L.csv ns 128 gather 4 > profiles/traffic_ns_n128_gather.json

One assembly step = the last `per_step` launches of the scatter's kernels
(gather: K2a + class kernel + the generic row launches)."""
import collections
import csv
import json
import sys


def main(path, config, n, scatter, per_step):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    K, M, V, I = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        launches.setdefault((int(r[I]), r[K]), {})[r[M]] = float(r[V].replace(",", ""))
    # the last complete step of this scatter's kernels (calibration runs of the
    # other scatter may follow in the list)
    prefix = "ff_gather" if scatter == "gather" else "ff_assemble"
    step = [kv for kv in launches.items() if kv[0][1].startswith(prefix)][-per_step:]
    kernels = [{"name": k, "dram_read": m["dram__bytes_read.sum"], "dram_write": m["dram__bytes_write.sum"],
                "ms": m["gpu__time_duration.sum"] / 1e6} for (_, k), m in step]
    out = {"config": config, "scatter": scatter,
           "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum ({path}), "
                     f"one assembly step = the last {per_step} ff_ launches",
           "kernels": kernels,
           "dram_bytes_per_launch": sum(k["dram_read"] + k["dram_write"] for k in kernels),
           "ms_serialised": sum(k["ms"] for k in kernels)}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4], int(sys.argv[5]))
