"""Synthetic benchmark inputs.

``synthetic_cifar10`` reproduces the reference's deterministic CIFAR-shaped
generator (``/root/reference/pkg/src/axemu/datasets.py:20-36``: ten 8x8-blocky
class templates from a fixed seed, 70% template + 30% uniform noise, snapped
to the byte grid) so benchmark batches are byte-identical to what the
reference harness would feed.  ``synthetic_imagenet`` is the same recipe at
224x224 (1000 blocky 7x7 class templates, each cell 32x32 pixels, 70% template
+ 30% uniform noise, byte grid): images with per-image global structure, so a
calibrated ResNet-50 predicts different classes for different images (plain
U[0,1) noise, ``uniform_images``, makes every image statistically identical
and every prediction the same).
"""

from __future__ import annotations

import numpy as np

_TEMPLATE_SEED = 20908


def class_templates() -> np.ndarray:
    base = np.random.default_rng(_TEMPLATE_SEED).uniform(0.0, 1.0, (10, 4, 4, 3))
    return base.repeat(8, axis=1).repeat(8, axis=2).astype(np.float32)


def synthetic_cifar10(n: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(seed)
    templates = class_templates()
    labels = rng.integers(0, 10, n)
    noise = rng.uniform(0.0, 1.0, (n, 32, 32, 3)).astype(np.float32)
    mixed = np.clip(0.7 * templates[labels] + 0.3 * noise, 0.0, 1.0)
    images = (np.rint(mixed * 255.0) / 255.0).astype(np.float32)
    return images, labels.astype(np.uint8)


def uniform_images(n: int, size: int = 224, seed: int = 0) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, 1.0, (n, size, size, 3)).astype(np.float32)


_IMAGENET_TEMPLATE_SEED = 20909


def synthetic_imagenet(n: int, seed: int = 0, size: int = 224) -> tuple[np.ndarray, np.ndarray]:
    """ImageNet-shaped synthetic batch: class template (7x7 cells of size/7 pixels) + 30% noise."""
    if size % 7:
        raise ValueError("size must be a multiple of 7")
    rng = np.random.default_rng(seed)
    labels = rng.integers(0, 1000, n)
    noise = rng.uniform(0.0, 1.0, (n, size, size, 3)).astype(np.float32)
    base = np.random.default_rng(_IMAGENET_TEMPLATE_SEED).uniform(0.0, 1.0, (1000, 7, 7, 3))
    cell = size // 7
    tmpl = base[labels].repeat(cell, axis=1).repeat(cell, axis=2).astype(np.float32)
    mixed = np.clip(0.7 * tmpl + 0.3 * noise, 0.0, 1.0)
    images = (np.rint(mixed * 255.0) / 255.0).astype(np.float32)
    return images, labels.astype(np.int64)
