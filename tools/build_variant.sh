# usage: bash tools/build_variant.sh <out.so> "<extra nvcc flags for fast_kernels.cu>"
# builds the library from the working tree in a scratch copy (the in-tree build is untouched)
set -e
out=$(realpath -m "$1"); extra="$2"
tmp=$(mktemp -d); mkdir -p $tmp/x/y
cp -r /root/repo/include $tmp/x/
cp -r /root/repo/paper_2403_12820_b200/csrc $tmp/x/y/
rm -rf $tmp/x/y/csrc/build
make -s -C $tmp/x/y/csrc -j4 FAST="--fmad=true -ftz=false $extra" > /dev/null
cp $tmp/x/y/libstencilcloth_b200.so "$out"
grep -A2 "fast_step_kernelILb1ELi4ELb0ELb0" $tmp/x/y/csrc/build/fast_kernels.ptxas.txt | grep -E "spill|Used" | tr '\n' ' '; echo
rm -rf $tmp
