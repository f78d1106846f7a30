# build HEAD's liblc into ab/old.so and the working tree's into ab/new.so (for scripts/ab.sh)
set -e
mkdir -p ab
rm -rf /tmp/wt_ab
git worktree add -f /tmp/wt_ab HEAD -q
(cd /tmp/wt_ab && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
   -Xcompiler -fPIC,-ffp-contract=off -shared -Iinclude -o "$OLDPWD/ab/old.so" paper_2603_17201_b200/csrc/*.cu)
git worktree remove --force /tmp/wt_ab
python -c "from paper_2603_17201_b200 import build; build.build()"
cp paper_2603_17201_b200/liblc.so ab/new.so
