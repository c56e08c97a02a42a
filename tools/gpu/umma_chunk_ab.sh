export TC_F32_UMMA=1
bash tools/gpu/ab_variants.sh "--only cfg4_ --reps 5" c4rna="-DTC_UMMA_HI_TRUNC=0" c2rna="-DTC_UMMA_HI_TRUNC=0 -DTC_UMMA_CHUNK=2" c1rna="-DTC_UMMA_HI_TRUNC=0 -DTC_UMMA_CHUNK=1" c2tr="-DTC_UMMA_CHUNK=2" c1tr="-DTC_UMMA_CHUNK=1" > gpurun_out/ab.txt 2>&1
python tools/f32_bias.py > gpurun_out/bias.jsonl 2>&1
for n in c4rna c2rna c1rna c2tr c1tr; do TC_B200_LIB=/tmp/tc_$n.so python tools/f32_bias.py >> gpurun_out/bias.jsonl 2>&1; done
