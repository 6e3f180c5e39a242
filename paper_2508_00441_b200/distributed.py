"""2-D output-tile sharding of one Ozaki DGEMM across the GPUs of a node.

C[I, J] depends only on A's row-panel I and B's column-panel J: slicing is
row-local for A and column-local for B (slicing.py:128-177) and the pair
order is per element (ozgemm.py:179-209).  So an R x Cc grid of ranks each
computes one C tile with the single-GPU kernels, bitwise identical to the
corresponding block of the 1-GPU result — there is no reduction on the hot
path.  The only collective is the one-time panel distribution: an NCCL
broadcast of A_I inside each row group and of B_J inside each column group
(NVLink / NVSwitch).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["TileGrid", "split_extent", "oz_gemm_tile"]


def split_extent(total: int, parts: int, idx: int) -> tuple[int, int]:
    """[lo, hi) of part idx when `total` is split into `parts` near-equal pieces
    (multiples of 128 where possible, so C tiles align with the 128x128 MMA tiles)."""
    if parts <= 0 or not 0 <= idx < parts:
        raise ValueError("bad partition")
    tiles = -(-total // 128)
    base, extra = divmod(tiles, parts)
    lo_t = idx * base + min(idx, extra)
    hi_t = lo_t + base + (1 if idx < extra else 0)
    return min(lo_t * 128, total), min(hi_t * 128, total)


@dataclass(frozen=True)
class TileGrid:
    rows: int  # R
    cols: int  # Cc

    @staticmethod
    def for_world(world: int) -> "TileGrid":
        """1 -> 1x1, 2 -> 1x2, 4 -> 2x2, 8 -> 2x4 (rows <= cols, as square as possible)."""
        r = int(world ** 0.5)
        while world % r:
            r -= 1
        return TileGrid(r, world // r)

    @property
    def size(self) -> int:
        return self.rows * self.cols

    def coords(self, rank: int) -> tuple[int, int]:
        return divmod(rank, self.cols)

    def rank_of(self, i: int, j: int) -> int:
        return i * self.cols + j

    def row_members(self, i: int):
        return [self.rank_of(i, j) for j in range(self.cols)]

    def col_members(self, j: int):
        return [self.rank_of(i, j) for i in range(self.rows)]

    def is_row_root(self, rank: int) -> bool:
        return self.coords(rank)[1] == 0

    def is_col_root(self, rank: int) -> bool:
        return self.coords(rank)[0] == 0

    def make_groups(self, dist):
        """Row and column process groups (every rank must call this, in order)."""
        rows = [dist.new_group(self.row_members(i)) for i in range(self.rows)]
        cols = [dist.new_group(self.col_members(j)) for j in range(self.cols)]
        return rows, cols

    def distribute_panels(self, dist, groups, rank: int, A_panel, B_panel) -> None:
        """Broadcast A_I from the row root along row group I and B_J from the
        column root along column group J (in place)."""
        i, j = self.coords(rank)
        rows, cols = groups
        if self.cols > 1:
            dist.broadcast(A_panel, src=self.rank_of(i, 0), group=rows[i])
        if self.rows > 1:
            dist.broadcast(B_panel, src=self.rank_of(0, j), group=cols[j])

    def tile_extent(self, rank: int, m: int, n: int):
        """Row range of A / C and column range of B / C owned by `rank`."""
        i, j = self.coords(rank)
        return split_extent(m, self.rows, i), split_extent(n, self.cols, j)


def oz_gemm_tile(A_panel, B_panel, cfg, out=None, graph: bool = False):
    """This rank's C tile C[I, J] = A_I @ B_J from its (distributed) panels with
    the single-GPU fused kernels — no reduction: slicing is row/column-local and
    the pair order is per element, so the tile is bitwise the single-GPU C's
    block.  Returns (C_tile, OzStats); used by bench.py's config-5 mode and the
    multi-rank GPU tests."""
    from .ozgemm import oz_gemm_device

    return oz_gemm_device(A_panel, B_panel, cfg, out=out, graph=graph)
