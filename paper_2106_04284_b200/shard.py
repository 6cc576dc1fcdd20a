"""Data-parallel extent sharding: the outermost array extent is
split into contiguous slabs, one per rank; each rank owns independent local
views (local extents) of its slab and relayouts them with no data-path
collective (every record's leaves are copied independently)."""


def shard_extents(extents, world, rank, multiple=1):
    """Returns (local_extents, first_record) for `rank` of `world`.

    Slab boundaries fall on whole rows of the outermost dimension and, when
    possible, on record indices that are multiples of `multiple` (e.g. the lcm
    of the AoSoA lane counts, so no block straddles two ranks).  For AoS and
    AoSoA layouts the concatenation of the local blobs is byte-identical to the
    global layout; for SoA each shard is its own SoA (reading #18)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    rows = int(extents[0])
    inner = 1
    for e in extents[1:]:
        inner *= int(e)
    step = 1  # rows per boundary quantum so that boundaries are multiples of `multiple` records
    while (step * inner) % multiple and step < rows:
        step += 1
    quanta = -(-rows // step)
    q0 = quanta * rank // world
    q1 = quanta * (rank + 1) // world
    r0 = min(rows, q0 * step)
    r1 = min(rows, q1 * step)
    return [r1 - r0] + [int(e) for e in extents[1:]], r0 * inner
