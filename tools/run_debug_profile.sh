# Build the event-log variant (libdmf_debug.so) and profile the asynchronous discharge.
set -e
export DMF_EXTRA_NVCC=-DDMF_DEBUG_BUSY
export DMF_LIB=$PWD/paper_2511_05895_b200/libdmf_debug.so
python -c "from paper_2511_05895_b200 import build as B; B.build()"
python tools/async_profile.py "$@"
