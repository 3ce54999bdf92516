# v7 ring-depth / poly sweep (build variants on the box)
for cfg in "3 2" "2 3" "2 2"; do
  set -- $cfg
  touch paper_2602_04789_b200/csrc/lfattn.cu
  LF_NVCC_FLAGS="-DLF_V7_KST=$1 -DLF_V7_VST=$2" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build fail $cfg"; continue; }
  for c in c2 c5_dense; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/v7_$1$2_$c.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/v7_$1$2_$c.json'));print('K$1 V$2 $c', round(d['value'],1), round(d['roofline']['achieved'],1))"
  done
done
touch paper_2602_04789_b200/csrc/lfattn.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c2 c5_dense; do
  LF_ATTN_POLY=4 timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/v7_poly4_$c.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/v7_poly4_$c.json'));print('POLY4 $c', round(d['value'],1), round(d['roofline']['achieved'],1))"
done
