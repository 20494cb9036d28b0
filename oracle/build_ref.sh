#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY.  Compiles the reference's own hot kernels
# (/root/reference/pkg/src/probegrid/backends/_core.pyx, Cython) from where
# they lie, with the reference's own compiler directives and flags
# (pkg/setup.py:27-43), into oracle/_ref/_core.<ext>.so.  Nothing from the
# reference is copied into the repository; only the built module lands in
# oracle/_ref/ (git-ignored, but shipped to the GPU box by gpurun).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src=/root/reference/pkg/src/probegrid/backends/_core.pyx
out="$here/_ref"
if [ ! -f "$src" ]; then
    echo "build_ref: $src not present; keeping prebuilt $out" >&2
    exit 0
fi
mkdir -p "$out"
ext="$(python3 -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
pyinc="$(python3 -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
stage_pkg() {
    # The reference package itself, staged (not committed: oracle/_ref is
    # git-ignored) so that -m gpu tests can drive the reference's OWN
    # orchestration (encoding.py, trainer.py, model_io.py) with this repo's
    # backend plugged into its seam (backends/__init__.py:12-50) on the GPU
    # box, where /root/reference does not exist.
    local pkg="$out/pkg"
    rm -rf "$pkg"
    mkdir -p "$pkg"
    cp -r /root/reference/pkg/src/probegrid "$pkg/probegrid"
    rm -f "$pkg/probegrid/backends/_core.pyx"
    find "$pkg" -name "__pycache__" -prune -exec rm -rf {} +
    cp "$out/_core$ext" "$pkg/probegrid/backends/_core$ext"
}
if [ -f "$out/_core$ext" ] && [ "$out/_core$ext" -nt "$src" ]; then
    [ -f "$out/pkg/probegrid/backends/_core$ext" ] || stage_pkg
    exit 0
fi
python3 -m cython -3 \
    -X boundscheck=False -X wraparound=False -X cdivision=True \
    -X initializedcheck=False \
    -o "$out/_core.c" "$src"
# -O3 without -march/-ffast-math exactly as pkg/setup.py:27-33
gcc -fno-strict-overflow -DNDEBUG -O3 -fPIC -fwrapv -I"$pyinc" \
    -shared -o "$out/_core$ext" "$out/_core.c"
rm -f "$out/_core.c"
echo "build_ref: built $out/_core$ext"
stage_pkg
