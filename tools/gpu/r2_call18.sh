set -x
mkdir -p gpurun_out/r2l
D=gpurun_out/r2l

export SAN_WORLD2=0 SAN_CASES=1,3 SAN_REFACTOR=1 DD_GRAPH=0 SAN_VARS=1,2,4,8,16,32,64,128,512,257,272
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool python tools/sanitize_target.py > $D/san_$tool.log 2>&1; tail -2 $D/san_$tool.log
done
