# build libtarragon from git revision $1 into /tmp/tg_ab/<rev>.so (A/B timing of code changes)
set -e
rev=$1
rm -rf /tmp/tg_ab_src && mkdir -p /tmp/tg_ab_src /tmp/tg_ab
git archive $rev include paper_2601_01310_b200 | tar -x -C /tmp/tg_ab_src
(cd /tmp/tg_ab_src && python paper_2601_01310_b200/build.py --force > /dev/null)
cp /tmp/tg_ab_src/paper_2601_01310_b200/libtarragon.so /root/repo/ab_$rev.so
echo /root/repo/ab_$rev.so
