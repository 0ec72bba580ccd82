# Build a diagnostic variant of the library with extra -D flags into build/variants/<name>/
#   bash tools/build_variant.sh fin2 -DICR_DIAG_FIN2
set -e
name=$1; shift
out=build/variants/$name; mkdir -p $out
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2603_13281_b200/csrc $*"
for f in paper_2603_13281_b200/csrc/*.cu; do nvcc $F -c $f -o $out/$(basename $f .cu).o & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart=static -o $out/libicarus_b200.so $out/*.o
echo $out/libicarus_b200.so
