"""Random-stream handle with the reference's addressing (reference samplers.py:122-147).

A stream is (seed, stream_id) plus a block cursor; every Philox4x32-10 block
yields two values and every request consumes whole blocks.  The engine's
device kernels (the dataset generator, `vb.vb_posterior_sample`) read the
stream at the cursor and advance it exactly as the reference would, so a
reference `tissuemix.samplers.RngStream` and this class are interchangeable
as arguments.
"""

from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class RngStream:
    seed: int
    stream_id: int = 0
    _block: int = field(default=0, repr=False)

    def spawn(self, stream_id: int) -> "RngStream":
        """Fresh stream under the same seed (reference samplers.py:145-147)."""
        return RngStream(self.seed, stream_id)

    def skip(self, n_values: int) -> None:
        """Advance past `n_values` values (ceil(n/2) blocks), as a draw of that size would."""
        self._block += -(-int(n_values) // 2)
