# A/B of hot-x packing variants (tools/exp_pack.py with variants/hot*.so)
for K in 8192 12288 16384 24576; do echo "== hot${K}na"; LWB200_LIB=variants/hot${K}na.so timeout 300 python tools/exp_pack.py 24 f32 $K; done
for K in 8192 16384; do echo "== hot${K}na f64"; LWB200_LIB=variants/hot${K}na.so timeout 300 python tools/exp_pack.py 24 f64 $K,-1; done
echo "== hot16384na s26"; LWB200_LIB=variants/hot16384na.so timeout 300 python tools/exp_pack.py 26 f32 16384,-1
