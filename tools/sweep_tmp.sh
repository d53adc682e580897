export DOT_TRAIN_LOCATE_LEVEL=7
bash tools/sweep_variants.sh l7 prod tools/variants/lib_m20.so tools/variants/lib_m16.so
