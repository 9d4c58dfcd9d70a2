"""The reference's tokenizer plug-in point (SessionConfig.tokenizer_encode /
tokenizer_decode, session.py:57-61, consumed at session.py:117-118,140,186,
227,336; contract SPEC.md:165):

    encode(GoP, CodecConfig) -> (TokenMatrix I, TokenMatrix P)
    decode(TokenMatrix I, TokenMatrix P, CodecConfig) -> GoP

A reference session runs its codec on the B200 with

    SessionConfig(..., tokenizer_encode=paper_2602_03529_b200.tokenizer_encode,
                       tokenizer_decode=paper_2602_03529_b200.tokenizer_decode)

The plug-in receives the already downscaled working GoP, exactly like the
reference's own encode_gop / decode_gop.
"""

from __future__ import annotations

from .codec import CodecConfig, TokenMatrix, decode_gop, encode_gop
from .video import GoP


def tokenizer_encode(gop: GoP, cfg: CodecConfig):
    return encode_gop(gop, cfg)


def tokenizer_decode(i_tokens: TokenMatrix, p_tokens: TokenMatrix, cfg: CodecConfig) -> GoP:
    return decode_gop(i_tokens, p_tokens, cfg)
