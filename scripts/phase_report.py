import re
import sys
buf = []
for l in open(sys.argv[1]):
    if l.startswith("family"):
        print(l.strip())
        for b in buf:
            d = dict(re.findall(r"(\w+)=(\d+)", b))
            dec = int(d["dec"])
            tot = sum(int(d[k]) for k in ["top", "carry", "arr", "score", "disp"])
            print("  dec", dec, "w1 %.2f w2 %.2f" % (int(d["w1"]) / dec, int(d["w2"]) / dec), "cyc/dec %.0f" % (tot / dec),
                  " ".join("%s %.0f" % (k, int(d[k]) / dec) for k in ["top", "carry", "arr", "score", "disp"]))
        buf = []
    elif l.startswith("PHASES"):
        buf.append(l)
