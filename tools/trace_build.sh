# Builds a phase-tracing variant of libkvlinc (-DKVLC_TRACE) into tools/_trace/.
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/_trace
for f in paper_2510_05373_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
       -diag-suppress 177 -DKVLC_TRACE -c "$f" -o "tools/_trace/$(basename "$f" .cu).o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/_trace/libkvlinc.so tools/_trace/*.o
