# build liblc with extra -D flags into ab/<name>.so:  bash scripts/build_variant.sh NAME -DFOO=1 ...
name=$1; shift
mkdir -p ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -shared "$@" -Iinclude -o ab/$name.so paper_2603_17201_b200/csrc/*.cu
