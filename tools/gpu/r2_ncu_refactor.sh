D=gpurun_out/rf
mkdir -p $D
timeout 300 python tools/ncu_refactor.py 5 > $D/plain.log 2>&1; cat $D/plain.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_refactor9 -s 1 -c 1 -o $D/prof_refactor9 -f python tools/ncu_refactor.py 2 > $D/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_blocks -s 2 -c 2 -o $D/prof_gather -f python tools/ncu_refactor.py 2 > $D/ncu2.log 2>&1
ls -la $D
