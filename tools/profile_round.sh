#!/bin/bash
# Round profile collection on the GPU box (run under gpurun; outputs under gpurun_out/):
#   bash tools/profile_round.sh r02b
# 1. the bench line, 2. the ncu launch list of the same bench command, 3. ncu --set full
# captures of the config kernels and of the cfg5 dense-A class (27 HBM-bound layers).
TAG=${1:-r02b}
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/${TAG}_bench_line.json 2> $OUT/${TAG}_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $OUT/${TAG}_launches_bench_cfg5.csv \
    python bench.py --steps 2 --warmup 3 > $OUT/${TAG}_ncu_bench.log 2>&1
for cfg in cfg2 cfg3a cfg3b cfg4; do
  ncu --set full --clock-control none --import-source on -k regex:igemm -s 3 -c 1 -f -o $OUT/${TAG}_${cfg}_full \
      python tools/prof_conv.py --config $cfg --iters 5 > $OUT/${TAG}_ncu_${cfg}.log 2>&1
done
DENSE=s1b1_1x1a,s1b1_1x1b,s1b1_proj,s1b2_1x1a,s1b2_1x1b,s1b3_1x1a,s1b3_1x1b,s2b1_1x1a,s2b1_1x1b,s2b2_1x1a,s2b2_1x1b,s2b3_1x1a,s2b3_1x1b,s2b4_1x1a,s2b4_1x1b,s3b1_1x1a,s3b1_1x1b,s3b2_1x1a,s3b2_1x1b,s3b3_1x1a,s3b3_1x1b,s3b4_1x1a,s3b4_1x1b,s3b5_1x1a,s3b5_1x1b,s3b6_1x1a,s3b6_1x1b
ncu --set full --clock-control none -k regex:igemm -c 27 -f -o $OUT/${TAG}_dense_class \
    python tools/prof_stack_layers.py --layers $DENSE --iters 1 > $OUT/${TAG}_ncu_dense.log 2>&1
IM2COL=s2b1_proj,s3b1_3x3,s3b1_proj,s3b2_3x3,s4b1_3x3,s4b1_proj,s4b2_3x3
ncu --set full --clock-control none -k regex:igemm -c 7 -f -o $OUT/${TAG}_im2col_class \
    python tools/prof_stack_layers.py --layers $IM2COL --iters 1 > $OUT/${TAG}_ncu_im2col.log 2>&1
# summaries (the reports themselves are too large to bring back: gpurun_out/ is capped at 64 MiB)
python tools/ncu_summary.py $OUT/${TAG}_cfg2_full.ncu-rep ${TAG}_cfg2_full cfg2_bf16_64x28x28x128_3x3 > /dev/null
python tools/ncu_summary.py $OUT/${TAG}_cfg3a_full.ncu-rep ${TAG}_cfg3a_full cfg3a_bf16_stem_32x224x224x3_7x7s2 > /dev/null
python tools/ncu_summary.py $OUT/${TAG}_cfg3b_full.ncu-rep ${TAG}_cfg3b_full cfg3b_bf16_16x64x64x256_3x3d2 > /dev/null
python tools/ncu_summary.py $OUT/${TAG}_cfg4_full.ncu-rep ${TAG}_cfg4_full cfg4_u8_128x28x28x256_3x3s2 > /dev/null
python tools/ncu_class_traffic.py $OUT/${TAG}_dense_class.ncu-rep "cfg5:icv_igemm_smem<bf16,dense>:hbm" ${TAG}_dense_class $DENSE
python tools/ncu_class_traffic.py $OUT/${TAG}_im2col_class.ncu-rep "cfg5:icv_igemm_smem<bf16,im2col>" ${TAG}_im2col_class $IM2COL
ncu -i $OUT/${TAG}_cfg4_full.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_cfg4_src.csv 2>/dev/null
python tools/ncu_source_top.py /tmp/${TAG}_cfg4_src.csv 25 > $OUT/${TAG}_cfg4_source_top.txt 2>&1
cp profiles/${TAG}_*.json profiles/ncu_traffic.json $OUT/
rm -f $OUT/*.ncu-rep
ls -la $OUT | grep $TAG
