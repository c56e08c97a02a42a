# red vs load-add-store, interleaved runs (order effects), f1 + f2 families
for pass in 1 2; do for v in nored def; do
  if [ $v = def ]; then LIB=""; else LIB=$PWD/build_var/lib_$v.so; fi
  TC_B200_LIB=$LIB timeout 900 python tools/suite.py --family f1 --no-ttdt > /tmp/f1_${v}_$pass.jsonl 2>/dev/null
  TC_B200_LIB=$LIB timeout 900 python tools/suite.py --family f2 --no-ttdt > /tmp/f2_${v}_$pass.jsonl 2>/dev/null
done; done
python - <<'PY'
import json
def load(v, p):
    d = {}
    for f in ("f1", "f2"):
        for l in open(f"/tmp/{f}_{v}_{p}.jsonl"):
            r = json.loads(l); d[r["config"]] = r["ms"]
    return d
runs = {(v, p): load(v, p) for v in ("nored", "def") for p in (1, 2)}
for k in runs[("def", 1)]:
    vals = [runs[(v, p)][k] * 1e3 for v in ("nored", "def") for p in (1, 2)]
    print(f"{k[:30]:30s} nored {vals[0]:8.1f} {vals[1]:8.1f}  red {vals[2]:8.1f} {vals[3]:8.1f}")
PY
