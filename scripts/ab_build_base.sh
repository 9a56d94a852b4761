# Build the library of a git revision (default HEAD) into
# paper_2306_08881_b200/lib/libacp_base.so for A/B runs (ACP_LIB=...).
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/acp_base && git -C "$ROOT" worktree prune && git -C "$ROOT" worktree add -f /tmp/acp_base "$REV" > /dev/null
python /tmp/acp_base/paper_2306_08881_b200/build.py > /dev/null
cp /tmp/acp_base/paper_2306_08881_b200/lib/libacp.so "$ROOT/paper_2306_08881_b200/lib/libacp_base.so"
git -C "$ROOT" worktree remove --force /tmp/acp_base
echo "base ($REV) -> paper_2306_08881_b200/lib/libacp_base.so"
