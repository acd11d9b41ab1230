#!/bin/bash
# ncu source capture of the 5/11 trio kernel for a library variant, reduced to tables.
#   scripts/ncu_one.sh variants/x.so tag   (run through gpurun for the capture part: MODE=capture)
set -e
lib=$1; tag=$2
if [ "$MODE" = capture ]; then
  HSAD_B200_LIB=$PWD/$lib ncu --set full --import-source on --clock-control none -k "regex:^detect_kernel$" -s 1 -c 1 \
    -o gpurun_out/$tag -f python scripts/probe_one.py 5 11 1 > gpurun_out/$tag.log 2>&1
  exit 0
fi
cd gpurun_out
ncu -i $tag.ncu-rep --page source --csv --print-source sass > $tag.sass.csv 2>/dev/null
mkdir -p x_$tag && cd x_$tag && cuobjdump -xelf detect.sm_100a.cubin ../../$lib > /dev/null && nvdisasm -gi -c detect.sm_100a.cubin > ../$tag.dis 2>/dev/null; cd ..
KN=$(grep -o '^_ZN[^:]*detect_kernelILi4ELi2ELi1ELb1ELb0ELb0ELb1E[^:]*' $tag.dis | head -1)
python ../scripts/sass_hotspots.py $tag.sass.csv $tag.dis "$KN" ../paper_1201_2025_b200/csrc/detect.cu | head -${HEAD:-30}
ncu -i $tag.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k in ['gpu__time_duration.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','launch__registers_per_thread']:
    print(k, v[h.index(k)])
"
