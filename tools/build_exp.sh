# experiment build of libgift (-DGIFT_SCAN_EXPERIMENT) -> tools/libgift_exp.so (never shipped)
set -e
cd "$(dirname "$0")/../paper_1604_01879_b200/csrc"
mkdir -p /tmp/expbuild
for f in util quantize fif_build fif_scan fif_scan_tc fif_scan_dense quant_tc topk act kmeans exact; do
  nvcc -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a \
    -DGIFT_SCAN_EXPERIMENT -c $f.cu -o /tmp/expbuild/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/libgift_exp.so /tmp/expbuild/*.o
