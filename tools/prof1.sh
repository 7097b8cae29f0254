set -x
NCU="ncu --set full --clock-control none --import-source on -k regex:k_tile_pass -s 1 -c 1"
timeout 300 $NCU -o gpurun_out/prof_x python tools/one_pass.py --kind X --targets 5,6,7,8 --n 40 --qubits 26 > /dev/null 2>&1
timeout 300 $NCU -o gpurun_out/prof_hlane python tools/one_pass.py --kind H --targets 0,1,2,3,4 --n 40 --qubits 26 > /dev/null 2>&1
timeout 300 $NCU -o gpurun_out/prof_h python tools/one_pass.py --kind H --targets 5,6,7,8 --n 40 --qubits 26 > /dev/null 2>&1
ls -la gpurun_out
