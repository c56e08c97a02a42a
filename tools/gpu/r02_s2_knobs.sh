# knob sweep on the fp64 stragglers: f2_16 (fig:bench ab-cad-dcb), cfg4_11 / cfg4_08 fp64
mkdir -p gpurun_out
run() {  # label, env..., family, case
  lab=$1; shift; fam=$1; shift; c=$1; shift
  env "$@" timeout 300 python tools/suite.py --no-ttdt --family $fam --only $c --reps 5 | sed "s/^/$lab /" >> gpurun_out/knobs.txt 2>&1
}
for rep in 1 2; do
  for c in f2_16 f2_17; do
    run def f2 $c X=1
    run now f2 $c TC_SK_WEIGHTS=0
    run msk4 f2 $c TC_WS_MINSK=4
    run msk16 f2 $c TC_WS_MINSK=16
    run msk32 f2 $c TC_WS_MINSK=32
    run csk16 f2 $c TC_CSK_MAX=16
    run nocsk f2 $c TC_CSK=0
  done
  for c in cfg4_11_f64 cfg4_08_f64 cfg4_04_f64; do
    run def baseline $c X=1
    run dp70 baseline $c TC_WS_DPPCT=70
    run dp95 baseline $c TC_WS_DPPCT=95
    run dp101 baseline $c TC_WS_DPPCT=101
    run gelem baseline $c TC_GATHER=elem
    run gmix baseline $c TC_GATHER=mixed
    run nows baseline $c TC_WAVE_SYNC=0
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(lambda: collections.defaultdict(list))
for l in open("gpurun_out/knobs.txt"):
    v, j = l.split(" ", 1)
    try: r = json.loads(j)
    except Exception: continue
    d[r["config"]][v].append((r["ms"], r["vs_gemm"]))
for c, x in d.items():
    print(c[:28], " ".join("%s %.4f(%.3f)" % (k, min(v)[0], max(w for _, w in v)) for k, v in x.items()))
PY
