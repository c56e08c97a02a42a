# build the default library and variants given as NAME=FLAGS pairs, run `suite.py ARGS` with each
# usage: bash tools/gpu/ab_variants.sh "<suite args>" name1="-DX=1" name2="-DY=2" ...
args=$1; shift
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python tools/suite.py --no-ttdt $args > gpurun_out/v_default.jsonl 2>&1
names="default"
for kv in "$@"; do
  n=${kv%%=*}; f=${kv#*=}
  TC_LIB_OUT=/tmp/tc_$n.so TC_NVCC_EXTRA="$f" python paper_1607_00291_b200/_build.py > /dev/null 2>&1 || echo "variant $n build failed"
  TC_B200_LIB=/tmp/tc_$n.so timeout 900 python tools/suite.py --no-ttdt $args > gpurun_out/v_$n.jsonl 2>&1
  names="$names $n"
done
python tools/compare_many.py $names
