L=paper_2508_00441_b200/liboz_b200.so
for r in 1 2; do for v in tf1 tf0; do cp liboz_$v.so $L; for n in 1024 2048; do timeout 300 python tools/ab_variant.py $n 1 | grep -v "(2, 192)\|(2, 128)" | sed "s/^/$v n=$n /"; done; timeout 300 python tools/k3_time.py $v; done; done
cp liboz_tf1.so $L
