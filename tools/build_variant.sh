# builds libkvlinc with extra nvcc defines into tools/_var/<name>/libkvlinc.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p tools/_var/$name
for f in paper_2510_05373_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
       -diag-suppress 177 "$@" -c "$f" -o "tools/_var/$name/$(basename "$f" .cu).o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/_var/$name/libkvlinc.so tools/_var/$name/*.o
