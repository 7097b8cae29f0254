for v in ${VARIANTS:-base}; do
if [ $v = base ]; then L=paper_1802_08032_b200/_lib/libqgpu.so; else L=paper_1802_08032_b200/_lib/libqgpu_$v.so; fi
echo "=== $v"
QGPU_LIB=$L timeout 300 python tools/sweep.py --kinds RZ,RY,X --counts 1,8,16,32 --targets 5,6,7
QGPU_LIB=$L timeout 300 python tools/sweep.py --kinds RY --counts 1,4,8,16 --targets 5,6,7,8,9,10,11
QGPU_LIB=$L timeout 300 python tools/sweep.py --kinds RY,X --counts 1,4,8,16 --targets 0,1,2,3,4
done
