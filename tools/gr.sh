# Local wrapper: rebuild every native artefact, then one gpurun call.
# usage: bash tools/gr.sh TIMEOUT_S 'command run on the GPU box'
set -e
T=$1; shift
make -C /root/repo/paper_2403_05676_b200/csrc -j8 > /tmp/gr_build.log 2>&1 || { tail -20 /tmp/gr_build.log; exit 1; }
make -C /root/repo/oracle > /tmp/gr_oracle.log 2>&1 || { tail -20 /tmp/gr_oracle.log; exit 1; }
cd /root/repo
/usr/local/graft/bin/gpurun --timeout "$T" -- "$@"
