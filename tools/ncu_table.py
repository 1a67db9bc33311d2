"""Print one row per kernel launch from an `ncu --metrics ... --csv` log."""
import collections
import csv
import sys


def main():
    for path in sys.argv[1:]:
        rows = [r for r in csv.reader(open(path)) if len(r) > 10]
        if not rows:
            continue
        hdr = rows[0]
        ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
        d = collections.OrderedDict()
        for r in rows[1:]:
            d.setdefault(r[ii], {"name": r[ki]})[r[mi]] = r[vi]
        print("==", path)
        for k, v in d.items():
            name = v.pop("name")
            if name.startswith(("void at::", "at::")):
                continue
            print(f"{name[:48]:48s}", " ".join(f"{m.split('.')[0][-22:]}={val}" for m, val in v.items()))


if __name__ == "__main__":
    main()
