#!/bin/bash
D=gpurun_out/${1:-asm}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-format-compare > $D/bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_assemble" -c 1 -o $D/asm300 python tools/spmv_ab.py 300 sym > $D/ncu_asm.log 2>&1
