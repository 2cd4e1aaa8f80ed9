"""B200-native FlexCTC hot path (arXiv 2508.07315): batched CTC beam search with NGPU-LM-style
n-gram shallow fusion and Aho-Corasick phrase boosting, as hand-written sm_100a CUDA behind a
C ABI (include/flexctc.h). See DESIGN.md."""
from .flexctc import (LM, Boost, Config, FlexCTCError, check, config, decode, decode_host, decode_host_bf16, decode_logits_bf16, decode_nbest, stats,  # noqa: F401
                      host_scratch_bytes, host_streaming, make_workspace, version, workspace_bytes)
