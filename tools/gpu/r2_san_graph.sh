# conditional-graph memcheck probe: minimal micro (tools/micro/cond_graph, no
# product code) and the product's two-context graph solve (tools/san_graph2.py)
mkdir -p gpurun_out/sg
D=gpurun_out/sg
tools/micro/cond_graph > $D/micro_plain.log 2>&1; echo "micro plain rc=$?" >> $D/micro_plain.log
timeout 300 compute-sanitizer --tool memcheck tools/micro/cond_graph > $D/micro_seq.log 2>&1; echo "rc=$?" >> $D/micro_seq.log
timeout 300 compute-sanitizer --tool memcheck tools/micro/cond_graph keep > $D/micro_keep.log 2>&1; echo "rc=$?" >> $D/micro_keep.log
KEEP=0 timeout 600 compute-sanitizer --tool memcheck python tools/san_graph2.py > $D/prod_seq.log 2>&1; echo "rc=$?" >> $D/prod_seq.log
KEEP=1 timeout 600 compute-sanitizer --tool memcheck python tools/san_graph2.py > $D/prod_keep.log 2>&1; echo "rc=$?" >> $D/prod_keep.log
for f in $D/*.log; do echo "== $f"; tail -n 12 $f; done
