L=paper_2508_00441_b200/liboz_b200.so
for r in 1 2 3; do for v in int0 int1; do cp liboz_$v.so $L; timeout 300 python tools/k3_time.py $v; done; done
cp liboz_int1.so $L
