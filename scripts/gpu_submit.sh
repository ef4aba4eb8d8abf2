# usage: bash scripts/gpu_submit.sh TIMEOUT_S SCRIPT [args...]
# Rebuilds every in-tree artefact HERE first (the snapshot ships the built .so
# files), then runs SCRIPT on a B200 through gpurun.
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()"
T=$1; shift
exec /usr/local/graft/bin/gpurun --timeout "$T" -- bash "$@"
