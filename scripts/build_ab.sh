# usage: bash scripts/build_ab.sh <git-rev> -- builds libmist.so of <rev> into ab/libmist_<rev>.so (A/B runs: MIST_LIB=...)
set -e
REV=${1:-HEAD}
WT=/tmp/mist_wt_$$
git -C /root/repo worktree add -f $WT $REV >/dev/null 2>&1
(cd $WT && python -m paper_2503_19050_b200.build --force >/dev/null 2>&1)
mkdir -p /root/repo/ab
cp $WT/paper_2503_19050_b200/libmist.so /root/repo/ab/libmist_$REV.so
git -C /root/repo worktree remove --force $WT
echo /root/repo/ab/libmist_$REV.so
