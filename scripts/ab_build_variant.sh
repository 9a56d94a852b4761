# Build HEAD + a patch into paper_2306_08881_b200/lib/libacp_NAME.so (A/B runs).
# usage: bash scripts/ab_build_variant.sh NAME PATCH
set -e
NAME=$1; PATCH=$(readlink -f "$2")
ROOT=$(cd "$(dirname "$0")/.." && pwd)
D=/tmp/acp_var_$NAME
rm -rf $D && git -C "$ROOT" worktree prune && git -C "$ROOT" worktree add -f $D HEAD > /dev/null
git -C $D apply "$PATCH"
python $D/paper_2306_08881_b200/build.py > /dev/null
cp $D/paper_2306_08881_b200/lib/libacp.so "$ROOT/paper_2306_08881_b200/lib/libacp_$NAME.so"
git -C "$ROOT" worktree remove --force $D
echo "$NAME -> paper_2306_08881_b200/lib/libacp_$NAME.so"
