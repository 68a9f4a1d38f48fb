# build variant: bv.sh name "flags"
name=$1; flags=$2
mkdir -p /tmp/irgl_vbuild/$name variants
for f in csrc/expand.cu csrc/topo.cu csrc/testops.cu csrc/gen.cu csrc/mst.cu csrc/relabel.cu csrc/api.cu; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -I../include -Icsrc --expt-relaxed-constexpr $flags -c $f -o /tmp/irgl_vbuild/$name/$(basename $f .cu).o || exit 1
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libirgl_rt_$name.so /tmp/irgl_vbuild/$name/*.o build/nccl_dyn.o build/frontend.o -ldl
