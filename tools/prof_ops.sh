# ncu source-level captures of single-config tile passes (26 qubits)
mkdir -p gpurun_out
cap() { name=$1; shift; timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_tile_pass -s 1 -c 1 -o gpurun_out/op_$name python tools/one_pass.py --qubits 26 "$@" > gpurun_out/op_$name.log 2>&1; echo $name=$?; }
cap ry32 --kind RY --targets 5,6,7 --n 32
cap lane32 --kind RY --targets 0,1,2 --n 32
cap cx32 --kind X --targets 5,6 --controls 7 --n 32
cap ry3ph --kind RY --targets 5,6,7,8,9,10,11 --n 14
timeout 300 python tools/sweep.py --kinds X,PHASE --counts 8,16,32 --targets 5,6 --controls 7
timeout 300 python tools/sweep.py --kinds X,PHASE --counts 8,16,32 --targets 5,6 --controls 2
timeout 300 python tools/sweep.py --kinds X,PHASE --counts 8,16,32 --targets 5,6 --controls 20
